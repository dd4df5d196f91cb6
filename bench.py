"""Benchmark: MDP build + value-iteration solve (BASELINE.json metric).

One step = the planner's hot path on the paper-scale workload (C2:
100x100x100 grid, 16 actions, 5000 DO realizations, time objective):
exact sub-grid sizing (k_vmax) + model build (k_build) + backward solve
(k_solve_layer), i.e. the reference's compute_subgrid + build_model +
value_iteration (pipeline.py:96-136) without file I/O.

  value : transitions/s = U / step time, U = N_c * nt * |A| * N_rv, inputs
          resident in HBM, device time (CUDA events), max over ranks.
  e2e   : the same metric through the public API from pinned HOST inputs:
          H2D of mean/modes/coeffs/g/mask + the step + D2H of everything the
          planner produces -- values, policy AND the compact transition model
          (row pointers, entry counts, rewards, entries).
  e2e_dropin : the reference callers' path (pipeline.run_build/run_solve
          without files): compute_subgrid + build_model -> host SparseModel
          (blocks[a][t] COO) + value_iteration(SparseModel) -> PolicyValue,
          host wall clock.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
With --gpus N > 1 and no torchrun environment, bench.py re-launches itself
under torch.distributed.run with N ranks (one per GPU).  Source rows are
split into y-strips (one per rank), the solve exchanges a one-sub-grid-wide
halo of V_{t+1} per layer over NCCL (strong scaling of the fixed C2 problem).

--impl reference: the reference's CPU path on the host cores (rank 0 only):
the oracle port (oracle/flowmdp_oracle.c) on a stratified sample -- every
source row of slabs t in {0, nt/3, 2nt/3}, scan + build + value iteration
-- each step; plus, once, the unmodified numpy reference (baseline/_ref) on
a realization-cropped sample at 1 process and at all cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "paper"


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default=WORKLOAD)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--reward-sum", default="sequential", choices=["sequential", "counts"],
                   help="row rewards: the reference's sequential sum (bit-exact, default) or formed from the "
                        "per-slot counts (rewards within ~1e-13 relative; north_star tolerance 1e-5)")
    p.add_argument("--reserve-sms", type=int, default=2,
                   help="SMs the build leaves to the pipelined solve stream (with --groups > 1)")
    p.add_argument("--upload-slabs", type=int, default=8,
                   help="end-to-end path: time slabs of the host->device upload, each scanned as soon as it lands")
    p.add_argument("--group-ratio", type=float, default=0.6,
                   help="slab group k (launch order, highest t first) holds a share of the slabs proportional "
                        "to ratio**k: < 1 shrinks the groups toward t = 0, so less of the solve and of the "
                        "model's D2H is left after the last group's build")
    p.add_argument("--groups", type=int, default=6,
                   help="slab groups per build: the solve of a group (and its halo exchange) and the model's "
                        "D2H start while the next group builds")
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                   help="gloo: validation of the N>1 path with several ranks on one GPU (halo and maxima "
                        "staged through host memory); never a bench number")
    return p.parse_args()


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._proc = None

    def __enter__(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for name, val in zip(names, r[3:]):
                if val.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU baselines (oracle/cpu_sample.py): the reference's CPU path on host cores
# ---------------------------------------------------------------------------

def _cpu_sample_mod():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import cpu_sample
    return cpu_sample


def config_of(w, world: int, backend: str = "nccl") -> dict:
    """The workload description both arms print (same keys, same values)."""
    g = w.grid
    return {"workload": w.name, "grid": [g.nx, g.ny, g.nt], "actions": w.n_actions,
            "realizations": w.n_realizations, "modes": w.n_modes, "objective": w.objective,
            "transitions": w.transitions,
            "parallelism": f"ystrips{world}" + ("-gloo-validation" if backend == "gloo" else ""),
            "l2": "flushed between steps (256 MiB write); inputs 185 MB > L2"}


def config_with_rewards(cfg: dict, reward_sum: str) -> dict:
    if reward_sum != "sequential":
        cfg = dict(cfg, reward_sum=reward_sum + " (rewards within 1e-12 relative of the sequential sum; "
                                               "counts / columns bit-exact)")
    return cfg


def cpu_baseline(w, env, subgrid=None) -> dict:
    """One stratified oracle-port step on every host core (the GPU arm's
    cpu_baseline: rank 0, N=1)."""
    CS = _cpu_sample_mod()
    threads = os.cpu_count() or 1
    r = CS.port_step(w, env, threads, subgrid=subgrid or w.subgrid_hint)
    return {"value": r["units"] / r["seconds"], "unit": "transitions/s", "cores": r["threads"], "kind": "port",
            "sample": CS.port_description(r, w), "seconds": r["seconds"],
            "full_step_s_extrapolated": r["full_step_s_extrapolated"]}


def run_reference(args):
    """The reference arm: rank 0 only (other ranks exit without work).

    Each of the W + K steps is one sampled planner step of the oracle port
    (scan + build + value iteration of three stratified slabs, all rows, all
    realizations, all host cores); the line's value is the transitions/s of
    the K timed steps.  ms_per_step is the measured duration of a step (of
    the sample); the full-step time is extrapolated separately and says so.
    The unmodified numpy reference is timed once on a smaller sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2109_00857_b200 import workloads
    CS = _cpu_sample_mod()
    w = workloads.get(args.workload)
    env = w.environment()
    threads = os.cpu_count() or 1
    runs = []
    for it in range(args.warmup + args.steps):
        r = CS.port_step(w, env, threads, subgrid=w.subgrid_hint)
        if it >= args.warmup:
            runs.append(r)
    units = sum(r["units"] for r in runs)
    seconds = sum(r["seconds"] for r in runs)
    value = units / seconds
    numpy_ref = None
    try:
        numpy_ref = CS.numpy_reference(w, env, ROOT)
    except Exception as exc:   # the supplementary numbers never fail the arm
        numpy_ref = {"error": f"{type(exc).__name__}: {exc}"}
    line = {
        "impl": "reference", "metric": "transitions_per_s", "value": value, "unit": "transitions/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": seconds / len(runs) * 1e3,
        "ms_per_step_note": "measured duration of one sampled step (3 of nt slabs, every row); not extrapolated",
        "full_step_ms_extrapolated": value and w.transitions / value * 1e3, "extrapolated_keys": ["full_step_ms_extrapolated"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(w, args.gpus, args.dist_backend),
        "stages_s_median": {k: statistics.median(r[k] for r in runs) for k in ("scan_s", "build_s", "vi_s")},
        "cpu_baseline": {"value": value, "unit": "transitions/s", "cores": runs[0]["threads"], "kind": "port",
                         "sample": CS.port_description(runs[0], w)},
        "numpy_reference": numpy_ref,
        "e2e": {"value": value, "unit": "transitions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def _load_json(path):
    try:
        return json.load(open(path))
    except Exception:
        return None


def hbm_peak_gbs():
    mp = _load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    for key in ("hbm_gbs", "hbm_gbps", "hbm_GBps", "hbm_copy_gbps", "hbm_burst_gbps"):
        if key in mp:
            return float(mp[key]), f"MEASURED_PEAKS.json:{key}"
    return 6650.0, "B200_PROFILING.md fallback (no HBM figure in MEASURED_PEAKS.json)"


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2109_00857_b200 as fm
    from paper_2109_00857_b200 import _lib, workloads
    from paper_2109_00857_b200.builder import DeviceEnv
    from paper_2109_00857_b200.sharding import StripPlanner, all_reduce_max, all_reduce_sum

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dist_backend == "gloo":   # ranks may share a GPU
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    L = _lib.load()
    s = _lib.stream_ptr()

    w = workloads.get(args.workload)
    env = w.environment()
    acts, rcfg = w.actions(), w.reward_config()
    g = w.grid

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        all_reduce_max(t)
        return float(t.item())

    # ---- device-resident step -------------------------------------------------
    # one process per GPU; the y-strips are cut by estimated build cost; at
    # N > 1 the build runs in 5 descending slab groups with the per-layer
    # solve + halo exchange of each group pipelined on a second stream
    denv = DeviceEnv.from_host(env)
    planner = StripPlanner(denv, acts, rcfg, w.target, w.buffer, n_groups=args.groups,
                           reserve_sms=args.reserve_sms if args.groups > 1 else 0, reward_sum=args.reward_sum,
                           group_ratio=args.group_ratio)
    j0, j1 = planner.j0, planner.j1
    n_g = g.nx * g.ny * g.nt
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    stages = []

    def step(de, scanned=False):
        planner.denv = de
        dm = planner.step(scanned=scanned)
        stages.append(dict(planner.events, nnz=dm.nnz))
        return dm

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        step(denv)
    torch.cuda.synchronize()
    stages.clear()
    launches0 = L.fm_kernel_launches()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()   # L2 flush between timed steps (inputs also exceed L2)
            barrier()
            torch.cuda.synchronize()
            e0, e1 = ev(), ev()
            e0.record()
            dm = step(denv)
            e1.record()
            torch.cuda.synchronize()
            barrier()
            times.append(e0.elapsed_time(e1))
        launches = (L.fm_kernel_launches() - launches0) // args.steps
        total_ms = max_over_ranks(sum(times))
        ms_per_step = total_ms / args.steps
        value = w.transitions / (ms_per_step / 1e3)
        build_ms = statistics.median(e["start"].elapsed_time(e["built"]) for e in stages)
        scan_ms = statistics.median(e["start"].elapsed_time(e["scanned"]) for e in stages)
        kbuild_ms = statistics.median(e["scanned"].elapsed_time(e["built"]) for e in stages)
        solve_ms = statistics.median(e["built"].elapsed_time(e["solved"]) for e in stages)
        nnz_rank = stages[-1]["nnz"]

        # ---- end to end through the public API, pinned host buffers ----------
        pinned = {
            "mean": torch.from_numpy(np.ascontiguousarray(env.field.mean)).pin_memory(),
            "modes": torch.from_numpy(np.ascontiguousarray(env.field.modes)).pin_memory(),
            "coeffs": torch.from_numpy(np.ascontiguousarray(env.field.coeffs)).pin_memory(),
            "g": torch.from_numpy(np.ascontiguousarray(env.scalar.g_mean)).pin_memory(),
            "mask": torch.from_numpy(env.obstacles.mask.view(np.uint8)).pin_memory(),
        }

        class _HostEnv:   # the reference's Environment shape, backed by pinned tensors
            grid = g
            field = type("F", (), {"mean": pinned["mean"], "modes": pinned["modes"], "coeffs": pinned["coeffs"]})()
            scalar = type("S", (), {"g_mean": pinned["g"]})()
            obstacles = type("O", (), {"mask": pinned["mask"]})()

        h2d = sum(t.numel() * t.element_size() for t in pinned.values())
        host_v = torch.empty(n_g + 1, dtype=torch.float64).pin_memory()
        host_p = torch.empty(n_g, dtype=torch.int16).pin_memory()
        # the compact transition model comes out too (north_star: "transition
        # model plus value function and policy out"): this rank's row
        # pointers, entry counts, rewards (strip-local, contiguous) and its
        # entries, on a copy stream that overlaps the solve
        # streamed group by group while the build runs (DeviceModel.stream_to_host)
        host_m = planner.dm.host_buffers()
        d2h_stream = torch.cuda.Stream()
        e2e_times, d2h_counts = [], []
        for it in range(args.warmup + args.steps):
            flush.zero_()
            barrier()
            torch.cuda.synchronize()
            e0, e1 = ev(), ev()
            e0.record()
            # upload in time slabs, the exact sub-grid scan of each slab
            # overlapping the next slab's copy (the planner's host-input path)
            de = DeviceEnv.from_host_scanned(_HostEnv, slabs=args.upload_slabs, j_range=(j0, j1) if world > 1 else None)
            planner.denv = de
            dm = planner.step(scanned=True, sink=host_m, sink_stream=d2h_stream)
            stages.append(dict(planner.events, nnz=dm.nnz))
            nbytes = planner.sink_bytes
            lo, hi = j0 * g.nx, j1 * g.nx
            if world == 1:
                host_v.copy_(planner.values, non_blocking=True)
                host_p.copy_(planner.policy, non_blocking=True)
                nbytes += (n_g + 1) * 8 + n_g * 2
            else:
                for t_ in range(g.nt):   # this rank's strip of every layer
                    a_, b_ = t_ * g.nx * g.ny + lo, t_ * g.nx * g.ny + hi
                    host_v[a_:b_].copy_(planner.values[a_:b_], non_blocking=True)
                    host_p[a_:b_].copy_(planner.policy[a_:b_], non_blocking=True)
                nbytes += (hi - lo) * g.nt * (8 + 2)
            torch.cuda.current_stream().wait_stream(d2h_stream)
            e1.record()
            torch.cuda.synchronize()
            barrier()
            if it >= args.warmup:
                e2e_times.append(e0.elapsed_time(e1))
                d2h_counts.append(nbytes)
        e2e_ms = max_over_ranks(sum(e2e_times))
        d2h = int(statistics.median(d2h_counts))
        if world > 1:
            t = torch.tensor([float(d2h)], dtype=torch.float64, device="cuda")
            all_reduce_sum(t)
            d2h_total = int(t.item())
        else:
            d2h_total = d2h
        e2e_value = w.transitions / (e2e_ms / args.steps / 1e3)
    clocks = clk.summary()

    # ---- the reference callers' drop-in path (world 1: a host SparseModel) ----
    dropin = None
    if world == 1:
        from paper_2109_00857_b200 import StepContext
        dts = []
        for it in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx = StepContext(env, acts, rcfg, w.target)
            sub = fm.compute_subgrid(env.field, acts, g, buffer=w.buffer, device_env=ctx.device_env())
            sm = fm.build_model(ctx, sub)
            pv = fm.value_iteration(sm)
            dts.append(time.perf_counter() - t0)
            del sm, ctx
        dt_ = statistics.median(dts[1:])
        dropin = {"value": w.transitions / dt_, "unit": "transitions/s", "ms_per_step": dt_ * 1e3,
                  "path": "StepContext -> compute_subgrid -> build_model -> host SparseModel (blocks[a][t] COO, "
                          "f64 vals) -> value_iteration(SparseModel) (Jacobi, reference semantics) -> PolicyValue; "
                          "host wall clock, numpy inputs (pageable), 1 warm-up + 2 timed",
                  "jacobi_iterations": pv.iterations_run, "residual": pv.residual}

    # ---- roofline of the dominant kernel (k_build) ------------------------------
    # algorithmic work F = 13 + 4 N_m / |A| flops per
    # transition (the reference's per-transition arithmetic), achieved =
    # U F / t_build, against the peak of the pipe the build actually uses --
    # "FP32 if the filtered FP32 path is adopted" (the binned build: one f32
    # reconstruction + bucket per (cell, realization), exact f64 only for the
    # realizations near a landing step).  t_build = the k_build launches alone
    # (CUDA events between the scan and the end of the build, on the stream
    # the kernels run on).  The executed f32 work and the issue-slot use of
    # the same launches are reported beside it.
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    f_clk = (clocks["sm_mhz"] or 1965.0) * 1e6
    cells_rank = (j1 - j0) * g.nx
    units_rank = cells_rank * g.nt * w.n_actions * w.n_realizations
    F = 13 + 4 * w.n_modes / w.n_actions
    achieved = units_rank * F / (kbuild_ms / 1e3)
    fp32_peak = sm_count * 128 * 2 * f_clk
    cell_real = cells_rank * g.nt * w.n_realizations
    flops_cr = 4 * w.n_modes + 8
    prof = _load_json(os.path.join(ROOT, "profiles", "r02d_k_build_paper_ncu.json")) or {}
    traffic = prof.get("dram_bytes_build") if args.workload == WORKLOAD else None
    issue = None
    if prof.get("warp_instructions_build") and args.workload == WORKLOAD and world == 1:
        ach_i = prof["warp_instructions_build"] / (kbuild_ms / 1e3)
        issue = {"achieved": ach_i / 1e12, "peak": sm_count * 4 * f_clk / 1e12, "unit": "Twarp-instr/s",
                 "frac": ach_i / (sm_count * 4 * f_clk),
                 "note": "ncu executed warp instructions of one build (profiles/r02d_k_build_paper_ncu.json) / "
                         "this run's k_build time, against 4 issue slots per SM per clock"}
    fp64_ceiling = sm_count * 64 * f_clk

    # backward solve against HBM: 12 B per entry (4 B column
    # + 8 B probability), 8 B reward per (state, action) row, 18 B per state
    n_rows_rank = cells_rank * g.nt * w.n_actions
    solve_bytes = 12 * nnz_rank + 8 * n_rows_rank + 18 * cells_rank * g.nt
    hbm_peak, hbm_src = hbm_peak_gbs()

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            sg = planner.dm.subgrid
            cpu = cpu_baseline(w, env, subgrid=(sg.half_width_x, sg.half_width_y))
        line = {
            "metric": "transitions_per_s", "value": value, "unit": "transitions/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_with_rewards(config_of(w, world, args.dist_backend), args.reward_sum),
            "stages": {"scan_build_ms_median": build_ms, "scan_ms_median": scan_ms, "k_build_ms_median": kbuild_ms, "solve_exposed_ms_median": solve_ms,
                       "step_ms": ms_per_step, "nnz_rank0": nnz_rank, "strips": planner.bounds,
                       "pipelined_slab_groups": planner.n_groups,
                       "slab_group_ratio": planner.group_ratio},
            "e2e": {"value": e2e_value, "unit": "transitions/s", "h2d_bytes_per_step": h2d * world,
                    "d2h_bytes_per_step": d2h_total, "ms_per_step": e2e_ms / args.steps,
                    "path": "pinned host inputs -> DeviceEnv.from_host_scanned (slab-wise H2D + exact scan) -> "
                            "build in slab groups -> backward solve -> D2H of values, policy and the compact model "
                            "(row_ptr, row_nnz, reward, entries; streamed per slab group while later groups "
                            "build: DeviceModel.stream_to_host)"},
            "e2e_dropin": dropin,
            "roofline": {"bound": "fp32", "kernel": "k_build", "achieved": achieved / 1e12,
                         "peak": fp32_peak / 1e12, "unit": "TFLOP/s", "frac": achieved / fp32_peak,
                         "traffic": traffic, "ms_per_launch_set": kbuild_ms,
                         "flops_per_transition": F, "units_per_step": units_rank,
                         "peak_source": f"{sm_count} SMs x 128 FP32 lanes x 2 (FMA) x the median SM clock under "
                                        "load (no FP32 figure in MEASURED_PEAKS.json)",
                         "definition": "SURVEY.md 8(d): U x F / t_build, F = 13 + 4 N_m/|A| algorithmic flops per "
                                       "transition, P = the pipe the build uses (FP32: the filtered binned path)",
                         "traffic_note": "dram__bytes_read+write of the k_build launches of one build (ncu --set "
                                         "full), vs 185 MB of inputs + the emitted model"},
            "executed_roofline": {
                "achieved": cell_real * flops_cr / (kbuild_ms / 1e3) / 1e12, "peak": fp32_peak / 1e12,
                "unit": "TFLOP/s", "frac": cell_real * flops_cr / (kbuild_ms / 1e3) / fp32_peak,
                "flops_per_cell_realization": flops_cr,
                "note": "the f32 work the binned build executes: per (cell, realization) 2 N_m FMA per velocity "
                        "component + floor/frac/bucket (4 ops per component); the rest of its instructions are "
                        "integer binning and shared-memory counters -- see issue_roofline"},
            "issue_roofline": issue,
            "fp64_issue_ceiling_tflops": fp64_ceiling / 1e12,
            "solve_roofline": {"bound": "hbm", "kernel": "k_solve_layer (backward sweep, nt launches)",
                               "achieved": solve_bytes / (solve_ms / 1e3) / 1e9 if solve_ms > 0 else None,
                               "peak": hbm_peak, "unit": "GB/s",
                               "frac": solve_bytes / (solve_ms / 1e3) / 1e9 / hbm_peak if solve_ms > 0 else None,
                               "bytes_algorithmic": solve_bytes, "ms_exposed": solve_ms, "peak_source": hbm_src,
                               "note": "nt dependent layers (latency-bound); at N > 1 all but the last slab "
                                       "group's layers run under the build, so only the exposed part is timed"},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def spawn(args) -> int:
    """--gpus N > 1 without a torchrun environment: re-launch this script
    under torch.distributed.run with N ranks on this node."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = _args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
