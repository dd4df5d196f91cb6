"""dev: repeated C2 builds -- entry census and row_nnz stats must not vary."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2109_00857_b200 import workloads
from paper_2109_00857_b200.builder import DeviceEnv, build_device_model, subgrid_from_vmax
w = workloads.get(sys.argv[1] if len(sys.argv) > 1 else "paper")
env = w.environment()
de = DeviceEnv.from_host(env)
sub = subgrid_from_vmax(de.velocity_max(), w.f_max, env.grid)
res = []
for it in range(int(os.environ.get("REPS", 4))):
    dm = build_device_model(de, w.actions(), w.reward_config(), w.target, sub)
    dm.check()
    rn = dm.row_nnz.to(torch.int64) & 0xFFFF
    res.append((dm.nnz, int(rn.max()), float(dm.reward.sum())))
print(os.environ.get("TAG", ""), res, "OK" if len(set(res)) == 1 else "NONDETERMINISTIC")
