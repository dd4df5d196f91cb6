"""Summarise an ncu report: key SOL/occupancy metrics + hottest SASS lines."""
import csv, io, subprocess, sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "k_build"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40


def run(args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
hdr = rows[0]
ki, mn, mu, mv = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
want = ["Duration", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Active Warps Per SM", "Theoretical Active Warps per SM", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput",
        "Eligible Warps Per Scheduler", "No Eligible", "Dynamic Shared Memory Per Block", "Block Limit Registers",
        "Block Limit Shared Mem"]
seen = set()
for r in rows[1:]:
    if kern in r[ki] and r[mn] in want and r[mn] not in seen:
        seen.add(r[mn])
        print(f"{r[mn]:40s} {r[mv]} {r[mu]}")

src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                                        "--launch-count", "1", "--print-source", "sass"]))))
hdr = src[1]
data = []
for r in src[2:]:
    if len(r) != len(hdr) or r[0] == "Address":
        if data:
            break
        continue
    data.append(r)
f = lambda x: float(x.replace(",", "") or 0)
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(f(r[iex]) for r in data)
agg = {hdr[i]: sum(f(r[i]) for r in data) for i in stall}
s = sum(agg.values()) or 1
print("stalls:", [(k[6:], round(v / s * 100, 1)) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]])
print("total warp instructions", tot)
hot = sorted(data, key=lambda r: -f(r[iex]))[:top]
hot = sorted(hot, key=lambda r: int(r[ia], 16))
for r in hot:
    st = sorted(((f(r[i]), hdr[i][6:]) for i in stall), reverse=True)[:2]
    print(r[ia][-5:], f"{f(r[iex]) / tot * 100:5.2f}%", r[isrc][:60].ljust(60), [(n, int(v)) for v, n in st])
