"""Per-CUDA-line instruction / stall-sample shares of one kernel in an ncu
report (ncu --page source --print-source cuda,sass); dev tool.
usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [top]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
iex = h.index("Instructions Executed")
isamp = h.index("Warp Stall Sampling (All Samples)")
iwf = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else None
def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0
agg = defaultdict(lambda: [0.0, 0.0, 0.0, ""])
line = None
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    if r[0]:
        line = r[0]
        agg[line][3] = r[1].strip()
    a = agg[line]
    a[0] += f(r[iex]); a[1] += f(r[isamp]); a[2] += f(r[iwf]) if iwf is not None else 0
tot = sum(a[0] for a in agg.values()) or 1; ts = sum(a[1] for a in agg.values()) or 1
tw = sum(a[2] for a in agg.values()) or 1
print(f"total instr {tot:.3e}  samples {ts:.0f}  smem wavefronts {tw:.3e}")
for ln, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{ln:>5} instr {a[0]/tot*100:5.1f}%  samp {a[1]/ts*100:5.1f}%  wf {a[2]/tw*100:5.1f}%  {a[3][:80]}")
