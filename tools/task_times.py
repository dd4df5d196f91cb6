"""Per-task cycle counts of the obstacle launch (PART 2) of one build (needs a
-DFM_STATS library via FM_LIB_PATH; dev tool)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2109_00857_b200 import workloads, _lib
from paper_2109_00857_b200.builder import DeviceEnv, build_device_model, subgrid_from_vmax
name = sys.argv[1] if len(sys.argv) > 1 else "paper"
w = workloads.get(name)
env = w.environment()
de = DeviceEnv.from_host(env)
sub = subgrid_from_vmax(de.velocity_max(), w.f_max, env.grid)
L = _lib.load()
buf = (C.c_uint64 * (1 << 20))()
n = C.c_int32(0)
L.fm_dev_task_times(buf, 1 << 20, C.byref(n))
dm = build_device_model(de, w.actions(), w.reward_config(), w.target, sub)
torch.cuda.synchronize()
L.fm_dev_task_times(buf, 1 << 20, C.byref(n))
allb = np.frombuffer(buf, dtype=np.uint64)
a = allb[: n.value]
cnts = allb[1 << 18: (1 << 18) + 8 * n.value].reshape(-1, 8)
cyc = (a & ((1 << 36) - 1)).astype(np.float64)
path = (a >> 36) & 15
task = a >> 40
g = env.grid
groups = (g.nx * g.ny + 1) // 2
print(f"{name}: {n.value} obstacle tasks, total {cyc.sum() / 1.96e9 * 1e3:.1f} ms-warp, "
      f"mean {cyc.mean() / 1.96e3:.1f} us, p50 {np.median(cyc) / 1.96e3:.1f} us, p99 {np.percentile(cyc, 99) / 1.96e3:.1f} us, "
      f"max {cyc.max() / 1.96e3:.1f} us")
for pth in (0, 1, 2):
    m = path == pth
    if m.any():
        print(f"  path {pth} ({['legacy-only', 'binned', 'bin failed -> legacy'][pth]}): {m.sum()} tasks, "
              f"{cyc[m].sum() / 1.96e9 * 1e3:.1f} ms-warp, mean {cyc[m].mean() / 1.96e3:.1f} us, max {cyc[m].max() / 1.96e3:.1f} us")
top = np.argsort(-cyc)[:15]
for i in top:
    t, grp = int(task[i]) // groups, int(task[i]) % groups
    c0 = 2 * grp
    print(f"  task t={t} cells ({c0 % g.nx},{c0 // g.nx}),({(c0 + 1) % g.nx},{(c0 + 1) // g.nx}) path {int(path[i])} "
          f"{cyc[i] / 1.96e3:.1f} us  D {int(cnts[i,0])} gated {int(cnts[i,1])} pairs {int(cnts[i,2])} seg {int(cnts[i,3])} init {cnts[i,4]*64/1.96e3:.0f}us drain {cnts[i,5]*64/1.96e3:.0f}us loop+drain {cnts[i,6]*64/1.96e3:.0f}us pairs-loop {cnts[i,7]*64/1.96e3:.0f}us")
print("totals D, gated, pairs, seg:", cnts.sum(0)[:4], "init/drain/loop ms-warp", cnts.sum(0)[4:7] * 64 / 1.96e6)
