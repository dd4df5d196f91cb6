"""Quick timing probe of the planner stages on one workload (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_00857_b200 as fm
from paper_2109_00857_b200 import workloads
from paper_2109_00857_b200.builder import DeviceEnv, build_device_model, subgrid_from_vmax
from paper_2109_00857_b200.solver import solve_backward

name = sys.argv[1] if len(sys.argv) > 1 else "paper"
w = workloads.get(name)
t0 = time.time(); env = w.environment(); print("gen", time.time() - t0, flush=True)
acts, rcfg = w.actions(), w.reward_config()
denv = DeviceEnv.from_host(env)
torch.cuda.synchronize()
def ev(): return torch.cuda.Event(enable_timing=True)
res = []
for it in range(int(os.environ.get('QT_ITERS', 6))):
    denv.reset_derived()
    e0, e1, e2, e3 = ev(), ev(), ev(), ev()
    e0.record()
    vm = denv.velocity_max()
    e1.record()
    sub = subgrid_from_vmax(vm, acts.f_max, env.grid)
    dm = build_device_model(denv, acts, rcfg, w.target, sub)
    e2.record()
    v, p = solve_backward(dm)
    e3.record()
    torch.cuda.synchronize()
    res.append((e1.elapsed_time(e2), e0.elapsed_time(e1), e2.elapsed_time(e3)))
b = sorted(r[0] for r in res[1:])
print(f"{name} sub={sub} nnz={dm.nnz} build_ms min={b[0]:.2f} med={b[len(b)//2]:.2f} "
      f"vmax_ms={min(r[1] for r in res):.2f} solve_ms={min(r[2] for r in res):.2f} "
      f"trans/s={w.transitions/(b[0]/1e3):.3e}", flush=True)
