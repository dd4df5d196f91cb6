"""Instruction / stall-sample share per SASS address region of a kernel."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
gran = int(sys.argv[3], 0) if len(sys.argv) > 3 else 0x400
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
samp = hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][ia], 16)
tot = sum(f(r[iex]) for r in data); ts = sum(f(r[samp]) for r in data)
cur = None
for r in data:
    k = (int(r[ia], 16) - base) // gran
    if cur is None or cur[0] != k:
        if cur and (cur[1] / tot > 0.005 or cur[2] / ts > 0.005):
            print(f"{hex(cur[0]*gran):>8} instr {cur[1]/tot*100:5.1f}%  samples {cur[2]/ts*100:5.1f}%  first: {cur[3][:50]}")
        cur = [k, 0.0, 0.0, r[isrc].strip()]
    cur[1] += f(r[iex]); cur[2] += f(r[samp])
if cur and (cur[1] / tot > 0.005 or cur[2] / ts > 0.005):
    print(f"{hex(cur[0]*gran):>8} instr {cur[1]/tot*100:5.1f}%  samples {cur[2]/ts*100:5.1f}%  first: {cur[3][:50]}")
