"""Summarise an ncu --set full report of one planner step's kernels into
profiles/r02_k_build_<workload>_ncu.json (dev / evidence tool): per launch
duration (under ncu, cold, serialised), DRAM bytes, executed warp
instructions, issue-active %, pipe utilisation, occupancy, top stalls; plus
the build totals bench.py reads (dram_bytes_build, warp_instructions_build).
usage: python tools/build_profile_json.py REPORT OUT.json [note]"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units = r[0], r[1]
KEYS = {"gpu__time_duration.sum": "duration", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "smsp__inst_executed.sum": "warp_instructions",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_active_pct",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
        "launch__registers_per_thread": "registers", "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
        "launch__grid_size": "grid", "launch__block_size": "block",
        "launch__shared_mem_per_block_dynamic": "smem_per_block"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in h]
launches = []
for row in r[2:]:
    d = {"kernel": row[hdr.index("Kernel Name")]}
    for k, name in KEYS.items():
        if k in hdr:
            v, u = row[hdr.index(k)], units[hdr.index(k)]
            try:
                d[name] = float(v.replace(",", "")) * SCALE.get(u, 1)
            except ValueError:
                pass
    st = {}
    for i in stall_cols:
        try:
            st[hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(row[i].replace(",", ""))
        except ValueError:
            pass
    tot = sum(st.values()) or 1.0
    d["top_stalls_pct"] = {k: round(v / tot * 100, 1) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:6]}
    d["dram_bytes"] = d.get("dram_read", 0) + d.get("dram_write", 0)
    launches.append(d)
build = [d for d in launches if d["kernel"].startswith("void k_build") or d["kernel"].startswith("k_build")]
summary = {"report": rep.split("/")[-1], "note": note,
           "dram_bytes_build": sum(d["dram_bytes"] for d in build) if build else None,
           "warp_instructions_build": sum(d.get("warp_instructions", 0) for d in build) if build else None,
           "duration_s_build_under_ncu": sum(d.get("duration", 0) for d in build) if build else None,
           "launches": launches}
json.dump(summary, open(out, "w"), indent=1)
for d in launches:
    print(f"{d['kernel'][:40]:40s} {d.get('duration', 0) * 1e3:8.3f} ms  dram {d['dram_bytes'] / 1e6:8.1f} MB  "
          f"winstr {d.get('warp_instructions', 0):.3e}  issue {d.get('issue_active_pct', 0):5.1f}%  "
          f"fma {d.get('fma_pipe_pct', 0):5.1f}% alu {d.get('alu_pipe_pct', 0):5.1f}% lsu {d.get('lsu_pipe_pct', 0):5.1f}%  "
          f"warps {d.get('warps_active_pct', 0):5.1f}%  {d['top_stalls_pct']}")
