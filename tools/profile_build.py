"""One warm build of a workload, for ncu (-k regex:k_build -s 1 -c 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2109_00857_b200 import workloads
from paper_2109_00857_b200.builder import DeviceEnv, build_device_model, subgrid_from_vmax
from paper_2109_00857_b200.solver import solve_backward

name = sys.argv[1] if len(sys.argv) > 1 else "desk"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = workloads.get(name)
env = w.environment()
denv = DeviceEnv.from_host(env)
for _ in range(reps):
    denv.reset_derived()
    sub = denv.subgrid(w.f_max, w.buffer)   # the planner's path: envelope bounds (k_vmax<.., false>)
    dm = build_device_model(denv, w.actions(), w.reward_config(), w.target, sub)
    solve_backward(dm)
torch.cuda.synchronize()
print("done", name, dm.nnz)
