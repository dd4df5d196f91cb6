"""Per-phase device timeline of bench.py's step (dev tool): where the step
time goes between k_vmax, host work, k_build and the solve."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2109_00857_b200 import workloads
from paper_2109_00857_b200.builder import DeviceEnv, build_device_model, subgrid_from_vmax
from paper_2109_00857_b200.solver import solve_backward

w = workloads.get(sys.argv[1] if len(sys.argv) > 1 else "paper")
env = w.environment()
acts, rcfg, g = w.actions(), w.reward_config(), w.grid
de = DeviceEnv.from_host(env)
n_g = g.nx * g.ny * g.nt
values = torch.zeros(n_g + 1, dtype=torch.float64, device="cuda")
policy = torch.zeros(n_g, dtype=torch.int16, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)
for it in range(5):
    torch.cuda.synchronize()
    E = [ev() for _ in range(6)]
    W = []
    E[0].record(); W.append(time.perf_counter())
    de.reset_derived()
    vm = de.velocity_max(); W.append(time.perf_counter())
    E[1].record()
    sub = subgrid_from_vmax(vm, acts.f_max, g, w.buffer)
    dm = build_device_model(de, acts, rcfg, w.target, sub, defer_check=True); W.append(time.perf_counter())
    E[2].record()
    solve_backward(dm, values, policy); W.append(time.perf_counter())
    E[3].record()
    dm.check(); W.append(time.perf_counter())
    E[4].record()
    torch.cuda.synchronize(); W.append(time.perf_counter())
    d = [E[i].elapsed_time(E[i + 1]) for i in range(4)]
    print(f"it{it} dev: vmax+sync {d[0]:.2f}  build(enq) {d[1]:.2f}  solve(enq) {d[2]:.2f}  check {d[3]:.2f}  "
          f"total {E[0].elapsed_time(E[4]):.2f} ms | host: " +
          " ".join(f"{(W[i + 1] - W[i]) * 1e3:.2f}" for i in range(len(W) - 1)), flush=True)
