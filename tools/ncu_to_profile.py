"""Extract the judged metrics of one kernel from an ncu report into JSON.

usage: python tools/ncu_to_profile.py REPORT KERNEL_REGEX OUT.json [note]
"""
import csv, io, json, re, subprocess, sys

rep, kern, out = sys.argv[1], sys.argv[2], sys.argv[3]
note = sys.argv[4] if len(sys.argv) > 4 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units = r[0], r[1]
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1,
         "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1}
launches = []
for row in r[2:]:
    name = row[hdr.index("Kernel Name")]
    if not re.search(kern, name):
        continue
    d = {"kernel": name}
    for w in WANT:
        if w in hdr:
            v, u = row[hdr.index(w)], units[hdr.index(w)]
            try:
                x = float(v.replace(",", ""))
                d[w] = x * SCALE.get(u, 1) if u in SCALE else x
                d[w + ".unit"] = "byte" if "byte" in u else ("s" if "second" in u else u)
            except ValueError:
                d[w] = v
    launches.append(d)
if not launches:
    sys.exit(f"no launch of {kern} in {rep}")
first = launches[0]


def _sum_finite(ls):
    tot = 0.0
    for m in ls:
        b = m.get("dram__bytes_read.sum", float("nan")) + m.get("dram__bytes_write.sum", float("nan"))
        if not (b == b):   # a launch ncu could not replay: no total
            return None
        tot += b
    return tot
summary = {"report": rep.split("/")[-1], "kernel_regex": kern, "note": note, "launches": len(launches),
           "dram_bytes_per_launch": first.get("dram__bytes_read.sum", 0) + first.get("dram__bytes_write.sum", 0),
           "dram_bytes_all_launches": _sum_finite(launches),
           "fp64_pipe_pct_first": first.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
           "issue_active_pct_first": first.get("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
           "duration_s_under_ncu": first.get("gpu__time_duration.sum"), "metrics": launches}
def _clean(x):   # strict JSON: a launch ncu could not replay has NaN metrics
    if isinstance(x, float) and x != x:
        return None
    if isinstance(x, dict):
        return {k: _clean(v) for k, v in x.items()}
    if isinstance(x, list):
        return [_clean(v) for v in x]
    return x


json.dump(_clean(summary), open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in summary.items() if k != "metrics"}, indent=1))
