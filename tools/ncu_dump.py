"""Dump SASS lines with exec share for an address range of a kernel."""
import csv, io, subprocess, sys
rep, kern, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3], 0), int(sys.argv[4], 0)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
src = list(csv.reader(io.StringIO(out))); hdr = src[1]
data = []
for r in src[2:]:
    if len(r) != len(hdr) or r[0] == "Address":
        if data: break
        continue
    data.append(r)
f = lambda x: float(x.replace(",", "") or 0)
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
base = int(data[0][ia], 16)
tot = sum(f(r[iex]) for r in data)
for r in data:
    off = int(r[ia], 16) - base
    if lo <= off < hi and f(r[iex]) > 0:
        print(hex(off), f"{f(r[iex])/tot*100:6.3f}%", r[isrc].strip()[:80])
