"""C5 stress configuration on one B200 (dev / evidence tool).

400x400x200 grid, 32 actions, 10,000 DO realizations (1.024e13 transitions):
exact sub-grid scan + model build + backward solve on the device, timed with
CUDA events; then spot parity against the CPU oracle on slab x row-strip
samples (every row of every action, bit-exact), and size-independent checks
on the whole model (per-row counts sum to N_rv).  Prints one JSON line."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import torch
import oracle as O
from paper_2109_00857_b200 import workloads
from paper_2109_00857_b200.builder import DeviceEnv, build_device_model, subgrid_from_vmax
from paper_2109_00857_b200.solver import solve_backward

name = sys.argv[1] if len(sys.argv) > 1 else "stress"
w = workloads.get(name)
t0 = time.time()
env = w.environment()
gen_s = time.time() - t0
acts, rcfg, g = w.actions(), w.reward_config(), w.grid
de = DeviceEnv.from_host(env)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
res = []
dm = None
for it in range(2):
    de.reset_derived()
    torch.cuda.synchronize()
    e0, e1, e2, e3 = ev(), ev(), ev(), ev()
    e0.record()
    sub = de.subgrid(acts.f_max, w.buffer)   # envelope bounds (exact scan only if ambiguous)
    e1.record()
    dm = build_device_model(de, acts, rcfg, w.target, sub, defer_check=True, reuse=dm)
    e2.record()
    v, p = solve_backward(dm)
    e3.record()
    dm.check()
    torch.cuda.synchronize()
    res.append((e0.elapsed_time(e1), e1.elapsed_time(e2), e2.elapsed_time(e3), e0.elapsed_time(e3)))
vmax_ms, build_ms, solve_ms, step_ms = res[-1]
# per-row counts sum to N_rv over the whole model
ok_sum = True
per_layer = g.nx * g.ny * w.n_actions
for t in range(g.nt):
    rid = torch.arange(t * per_layer, (t + 1) * per_layer, device="cuda")
    ptr, cnt = dm.row_ptr[rid], dm.row_nnz[rid].to(torch.int64) & 0xFFFF
    seg = torch.repeat_interleave(torch.arange(per_layer, device="cuda"), cnt)
    idx = torch.repeat_interleave(ptr, cnt) + (torch.arange(int(cnt.sum()), device="cuda")
                                               - torch.repeat_interleave(torch.cumsum(cnt, 0) - cnt, cnt))
    c = dm.entries[idx].to(torch.int64) & 0xFFFF
    tot = torch.zeros(per_layer, dtype=torch.int64, device="cuda").index_add_(0, seg, c)
    ok_sum &= bool((tot == w.n_realizations).all().item())
# spot parity vs the oracle
checks = []
for t in (0, g.nt // 2, g.nt - 2, g.nt - 1):
    for (j0, j1) in ((0, 2), (g.ny // 2 - 1, g.ny // 2 + 1), (g.ny * 11 // 25, g.ny * 11 // 25 + 4)):
        om = O.build_model(env, acts, rcfg, w.target, sub.half_width_x, sub.half_width_y,
                           n_threads=os.cpu_count() or 1, t_range=(t, t + 1), j_range=(j0, j1))
        same = True
        for a in range(w.n_actions):
            r, c, vv, rew = dm.rows_coo(t, a, j0, j1)
            orr, oc, ov = om.blocks[a][t]
            n_g = g.nx * g.ny * g.nt
            ore = om.rewards[a * n_g + t * g.nx * g.ny + j0 * g.nx: a * n_g + t * g.nx * g.ny + j1 * g.nx]
            same &= (np.array_equal(r, orr) and np.array_equal(c, oc) and vv.tobytes() == ov.tobytes()
                     and rew.tobytes() == ore.tobytes())
        checks.append({"t": t, "rows": [j0, j1], "bit_exact": bool(same)})
out = {"workload": name, "grid": [g.nx, g.ny, g.nt], "actions": w.n_actions, "realizations": w.n_realizations,
       "transitions": w.transitions, "subgrid": [sub.half_width_x, sub.half_width_y], "nnz": dm.nnz,
       "vmax_ms": vmax_ms, "build_ms": build_ms, "solve_ms": solve_ms, "step_ms": step_ms,
       "transitions_per_s": w.transitions / (step_ms / 1e3), "build_transitions_per_s": w.transitions / (build_ms / 1e3),
       "device_mem_gb": torch.cuda.max_memory_allocated() / 1e9, "env_gen_s": gen_s,
       "v_start": float(v[g.state_index(*w.start, 0)].item()), "row_counts_sum_to_n_real": ok_sum,
       "oracle_spot_checks": checks}
print(json.dumps(out), flush=True)
