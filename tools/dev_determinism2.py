"""dev: which rows differ between repeated C2 builds."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2109_00857_b200 import workloads
from paper_2109_00857_b200.builder import DeviceEnv, build_device_model, subgrid_from_vmax
w = workloads.get(sys.argv[1] if len(sys.argv) > 1 else "paper")
env = w.environment()
de = DeviceEnv.from_host(env)
sub = subgrid_from_vmax(de.velocity_max(), w.f_max, env.grid)
g = env.grid
base = None
for it in range(4):
    dm = build_device_model(de, w.actions(), w.reward_config(), w.target, sub)
    dm.check()
    rn = (dm.row_nnz.to(torch.int64) & 0xFFFF).cpu()
    if base is None:
        base = rn
        continue
    d = torch.nonzero(rn != base).flatten()
    print("build", it, "differing rows", d.numel())
    for r in d[:12].tolist():
        a = r % 16; rc = r // 16; t = rc // (g.nx * g.ny); c = rc % (g.nx * g.ny)
        print(f"   row t={t} cell=({c % g.nx},{c // g.nx}) a={a} nnz {int(base[r])} vs {int(rn[r])}")
