"""dev: the drop-in build_model path at C2 -> SparseModel column range (+ A/B env)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2109_00857_b200 as fm
from paper_2109_00857_b200 import workloads, StepContext
w = workloads.get(sys.argv[1] if len(sys.argv) > 1 else "paper")
env, acts, rcfg = w.environment(), w.actions(), w.reward_config()
ctx = StepContext(env, acts, rcfg, w.target)
sub = fm.compute_subgrid(env.field, acts, env.grid, buffer=w.buffer, device_env=ctx.device_env())
from paper_2109_00857_b200.builder import build_device_model
dm = build_device_model(ctx.device_env(), acts, rcfg, w.target, sub)
rebuilt = dm.check()
print("nnz", dm.nnz, "rebuilt", rebuilt, "capacity", dm.entries.numel())
rn = dm.row_nnz.to(torch.int64) & 0xFFFF
print("row_nnz sum", int(rn.sum()), "max", int(rn.max()), "zero rows", int((rn == 0).sum()))
ent = dm.entries[: dm.nnz].to(torch.int64) & 0xFFFFFFFF
slot = ent >> 16
print("slot max", int(slot.max()), "nslot", (2 * sub.half_width_x + 1) * (2 * sub.half_width_y + 1))
sm = dm.to_sparse_model()
mx = max(int(b.cols.max()) for bl in sm.blocks for b in bl if b.nnz)
print("to_sparse_model: max col", mx, "n_states", sm.n_states)
sm2 = fm.build_model(ctx, sub)
mx = max(int(b.cols.max()) for bl in sm2.blocks for b in bl if b.nnz)
print("build_model: max col", mx, "n_states", sm2.n_states)
