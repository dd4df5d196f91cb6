"""Small builds + solves through every k_build path, for compute-sanitizer
(memcheck / racecheck / synccheck); dev / evidence tool.

Cases: lean cells binned (bin path, envelope and triangle bound), the
per-transition lean path (FM_NO_BINS), obstacle tasks with count-formed
rewards (deferred exact segment queue), net energy (in-place segment tests,
per-transition rewards), the fully checked path (lean=False) and the
global-histogram kernel (F_GHIST, huge sub-grid).  Each model is compared
with the oracle so a sanitizer run also proves the results."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np
import oracle as O
import paper_2109_00857_b200 as fm
from paper_2109_00857_b200 import workloads
from paper_2109_00857_b200.builder import DeviceEnv, build_device_model
from paper_2109_00857_b200.core_types import (ActionSpace, DOVelocityField, Environment, GridSpec, ObstacleMask,
                                              RewardConfig, ScalarMeanField)
from paper_2109_00857_b200.solver import solve_backward
from golden_util import model_digest


def check(name, env, acts, rcfg, target, **kw):
    denv = DeviceEnv.from_host(env)
    sub = fm.compute_subgrid(env.field, acts, env.grid, device_env=denv)
    if kw.pop("no_envelope", False):
        denv._env_rows = None
    dm = build_device_model(denv, acts, rcfg, target, sub, **kw)
    solve_backward(dm)
    om = O.build_model(env, acts, rcfg, target, sub.half_width_x, sub.half_width_y, n_threads=os.cpu_count() or 1)
    sm = dm.to_sparse_model()
    if kw.get("reward_sum") == "counts":   # counts / columns exact, rewards to rounding
        ok = all(np.array_equal(sm.blocks[a][t].cols, om.blocks[a][t][1]) and
                 sm.blocks[a][t].vals.tobytes() == om.blocks[a][t][2].tobytes()
                 for a in range(acts.n_actions) for t in range(env.grid.nt))
        ok = ok and float(np.max(np.abs(sm.rewards - om.rewards) / np.maximum(np.abs(om.rewards), 1.0))) <= 1e-12
    else:
        ok = model_digest(sm) == model_digest(om)
    print(f"{name}: {'bit-exact' if ok else 'MISMATCH'}", flush=True)
    assert ok


def small(name, n_rv=48, nt=6, **kw):
    w = workloads.get(name)
    w = w.with_(grid=GridSpec(nx=w.grid.nx, ny=w.grid.ny, nt=nt, dx=1.0, dt=1.0), n_realizations=n_rv, **kw)
    return w.environment(), w.actions(), w.reward_config(), w.target


which = sys.argv[1:] or ["bins", "bins_tri", "lean_pt", "obst", "obst_pt", "binonly_off", "net", "net_counts",
                         "checked", "ghist"]
for case in which:
    if case == "bins":
        check(case, *small("desk"))
    elif case == "bins_tri":
        check(case, *small("desk"), no_envelope=True)
    elif case == "lean_pt":
        os.environ["FM_NO_BINS"] = "1"
        check(case, *small("desk"))
        del os.environ["FM_NO_BINS"]
    elif case == "obst":   # obstacle tasks binned (bin-only launches + list launch)
        check(case, *small("paper_net_energy", objective="time"))
    elif case == "obst_pt":   # obstacle tasks per transition (deferred exact segment queue)
        os.environ["FM_NO_OBST_BINS"] = "1"
        check(case, *small("paper_net_energy", objective="time"))
        del os.environ["FM_NO_OBST_BINS"]
    elif case == "binonly_off":   # bins with the inline per-transition fallback (PART 1 / 2)
        os.environ["FM_NO_BINONLY"] = "1"
        check(case, *small("paper_net_energy", objective="time"))
        del os.environ["FM_NO_BINONLY"]
    elif case == "net_counts":
        check(case, *small("paper_net_energy"), reward_sum="counts")
    elif case == "net":
        check(case, *small("paper_net_energy"))
    elif case == "checked":
        check(case, *small("desk"), lean=False)
    elif case == "ghist":
        rng = np.random.default_rng(77)
        nx = ny = 72
        nt, nr, nm = 3, 40, 3
        g = GridSpec(nx=nx, ny=ny, nt=nt, dx=1.0, dt=1.0)
        mask = np.zeros((nt, ny, nx), dtype=bool)
        mask[:, 30:34, 20:26] = True
        env = Environment(grid=g, field=DOVelocityField(mean=rng.uniform(-30.0, 30.0, (nt, ny, nx, 2)),
                                                        modes=rng.normal(0, 0.4, (nm, nt, ny, nx, 2)),
                                                        coeffs=rng.normal(0, 0.5, (nt, nr, nm))),
                          scalar=ScalarMeanField(g_mean=rng.uniform(0, 2, (nt, ny, nx))),
                          obstacles=ObstacleMask(mask=mask))
        check(case, env, ActionSpace(8, 1, 1.0), RewardConfig("time", r_term=10.0, r_outbound=-30.0), (40, 40))
