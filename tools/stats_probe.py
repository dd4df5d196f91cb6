"""Path statistics of one build (needs a -DFM_STATS library via FM_LIB_PATH; dev tool)."""
import ctypes as C, os, sys
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
out = (C.c_uint64 * 8)()
L.fm_dev_stats(out)
dm = build_device_model(de, w.actions(), w.reward_config(), w.target, sub)
torch.cuda.synchronize()
L.fm_dev_stats(out)
names = ["rare", "seg_exact", "seg_samples", "obst_trans", "lean_trans", "bin_tasks", "bin_exact", "bin_misfit"]
print(name, {n: int(out[i]) for i, n in enumerate(names)}, "U", w.transitions)
