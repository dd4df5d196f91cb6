"""Randomised medium-size worlds through every build path, against the oracle.

The reference's random worlds (make_random_env) stay inside its dense
oracle's envelope (<= 64 cells, <= 64 realizations: one reconstruction chunk,
few obstacles).  These worlds are larger and stranger: several chunks per
task (80-300 realizations), arbitrary action counts (3-24: reconstruction lane
counts that do not divide a chunk, one to ten cells per warp), 0-9 modes,
random origin / dx / dt (so the F_PROVEN geometry is the general one and
F_CNT holds or not depending on dt), moving and random obstacles, every
objective; and some with a hand-shrunk sub-grid (the fully checked path and
its overflow report).  Every block, reward, value and action bit-exact."""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle as O
from golden_util import model_digest, sha

pytestmark = pytest.mark.gpu

fm = pytest.importorskip("paper_2109_00857_b200")
from paper_2109_00857_b200 import (  # noqa: E402
    ActionSpace,
    DOVelocityField,
    Environment,
    GridSpec,
    ObstacleMask,
    RewardConfig,
    ScalarMeanField,
    StepContext,
)
from paper_2109_00857_b200.builder import build_device_model  # noqa: E402
from paper_2109_00857_b200.solver import solve_backward  # noqa: E402


def fuzz_world(seed: int):
    rng = np.random.default_rng(seed)
    nx, ny, nt = int(rng.integers(6, 24)), int(rng.integers(6, 24)), int(rng.integers(4, 9))
    dx = float(rng.choice([0.25, 0.5, 1.0, 1.5, 3.0]))
    dt = float(rng.choice([0.3, 0.5, 1.0, 2.0]))
    origin = (float(rng.uniform(-40, 40)), float(rng.uniform(-40, 40)))
    g = GridSpec(nx=nx, ny=ny, nt=nt, dx=dx, dt=dt, origin=origin)
    nm, nr = int(rng.integers(0, 10)), int(rng.integers(80, 300))
    speed = dx / dt
    mean = rng.normal(0.0, 0.6 * speed, size=(nt, ny, nx, 2))
    modes = rng.normal(0.0, 1.0, size=(nm, nt, ny, nx, 2)) / np.sqrt(max(nx * ny, 1))
    coeffs = rng.normal(0.0, 0.8 * speed, size=(nt, nr, nm)) * np.sqrt(nx * ny) / max(nm, 1)
    mask = np.zeros((nt, ny, nx), dtype=bool)
    kind = seed % 3
    if kind == 0:   # a moving block
        for t in range(nt):
            i0 = (2 + t) % nx
            mask[t, ny // 3: ny // 3 + 3, i0: i0 + 3] = True
    elif kind == 1:   # scattered static cells
        mask[:] = rng.random((ny, nx)) < 0.1
    scalar = rng.uniform(0.0, 3.0, size=(nt, ny, nx))
    env = Environment(grid=g, field=DOVelocityField(mean=mean, modes=modes, coeffs=coeffs),
                      scalar=ScalarMeanField(g_mean=scalar), obstacles=ObstacleMask(mask=mask))
    n_h = int(rng.choice([3, 4, 5, 6, 7, 8, 12]))
    n_s = int(rng.choice([1, 2]))
    acts = ActionSpace(n_headings=n_h, n_speeds=n_s, f_max=float(rng.choice([0.5, 1.0])) * speed)
    obj = ("time", "energy", "net_energy")[seed % 3 if seed % 2 else (seed // 2) % 3]
    rcfg = RewardConfig(obj, c_f=float(rng.choice([1.0, 0.3])), c_r=0.6, r_term=float(rng.choice([50.0, 7.5])),
                        r_outbound=-120.0)
    while True:
        target = (int(rng.integers(0, nx)), int(rng.integers(0, ny)))
        if not mask[0, target[1], target[0]]:
            break
    return env, acts, rcfg, target


@pytest.mark.parametrize("seed", list(range(9000, 9040)))
def test_fuzz_world_parity(seed):
    env, acts, rcfg, target = fuzz_world(seed)
    ctx = StepContext(env, acts, rcfg, target)
    sub = fm.compute_subgrid(env.field, acts, env.grid)
    hx, hy = O.compute_subgrid(env.field, acts.f_max, env.grid)
    assert (sub.half_width_x, sub.half_width_y) == (hx, hy)
    gm = fm.build_model(ctx, sub)
    om = O.build_model(env, acts, rcfg, target, hx, hy, n_threads=os.cpu_count() or 1)
    assert model_digest(gm) == model_digest(om)
    denv = ctx.device_env()
    dmc = build_device_model(denv, acts, rcfg, target, sub, lean=False)   # fully checked path
    assert model_digest(dmc.to_sparse_model()) == model_digest(om)
    ov, oa, oit, ores, oconv = O.value_iteration(om)
    pv = fm.value_iteration(gm)
    assert sha(pv.values) == sha(ov) and sha(pv.actions) == sha(oa)
    assert (pv.iterations_run, pv.residual, pv.converged) == (oit, ores, oconv)
    if ores == 0.0:
        vals, pol = solve_backward(build_device_model(denv, acts, rcfg, target, sub))
        assert sha(vals.cpu().numpy()) == sha(ov)


@pytest.mark.parametrize("seed", list(range(9100, 9110)))
def test_fuzz_shrunk_subgrid(seed):
    """A sub-grid one cell narrower than compute_subgrid's: either the build
    fits (identical models) or both raise the same ContractViolation."""
    env, acts, rcfg, target = fuzz_world(seed)
    hx, hy = O.compute_subgrid(env.field, acts.f_max, env.grid)
    sub = fm.SubGridSpec(max(hx - 2, 0), max(hy - 2, 0))
    ctx = StepContext(env, acts, rcfg, target)
    try:
        om = O.build_model(env, acts, rcfg, target, sub.half_width_x, sub.half_width_y)
        ref_err = None
    except O.OracleViolation as exc:
        om, ref_err = None, str(exc)
    if ref_err is None:
        assert model_digest(fm.build_model(ctx, sub)) == model_digest(om)
    else:
        with pytest.raises(fm.ContractViolation) as ei:
            fm.build_model(ctx, sub)
        assert str(ei.value) == ref_err


def _edge_world(nx, ny, nt, nr, nm, n_h, n_s, mask_all_t1=False, seed=1):
    rng = np.random.default_rng(seed)
    g = GridSpec(nx=nx, ny=ny, nt=nt, dx=1.0, dt=1.0)
    mask = np.zeros((nt, ny, nx), dtype=bool)
    if mask_all_t1 and nt > 1:
        mask[1] = True
        mask[1, 0, 0] = False
    env = Environment(grid=g,
                      field=DOVelocityField(mean=rng.normal(0, 0.5, (nt, ny, nx, 2)),
                                            modes=rng.normal(0, 0.3, (nm, nt, ny, nx, 2)),
                                            coeffs=rng.normal(0, 0.5, (nt, nr, nm))),
                      scalar=ScalarMeanField(g_mean=rng.uniform(0, 2, (nt, ny, nx))),
                      obstacles=ObstacleMask(mask=mask))
    return env, ActionSpace(n_headings=n_h, n_speeds=n_s, f_max=1.0)


@pytest.mark.parametrize("case", [
    dict(nx=5, ny=4, nt=1, nr=7, nm=2, n_h=4, n_s=1),          # horizon layer only
    dict(nx=5, ny=4, nt=2, nr=1, nm=1, n_h=4, n_s=2),          # one realization
    dict(nx=1, ny=7, nt=4, nr=70, nm=3, n_h=4, n_s=1),         # one column
    dict(nx=9, ny=1, nt=4, nr=70, nm=0, n_h=8, n_s=1),         # one row, no modes
    dict(nx=6, ny=6, nt=4, nr=65, nm=8, n_h=1, n_s=1),         # a single action
    dict(nx=6, ny=6, nt=5, nr=64, nm=8, n_h=16, n_s=2, mask_all_t1=True),   # 32 actions, layer 1 all masked
    dict(nx=7, ny=5, nt=3, nr=129, nm=5, n_h=5, n_s=3),        # 15 actions, 3 chunks + 1
])
def test_edge_shapes(case):
    env, acts = _edge_world(**case)
    for obj, target in (("time", (0, 0)), ("net_energy", (env.grid.nx - 1, env.grid.ny - 1))):
        rcfg = RewardConfig(obj, c_f=1.0, c_r=0.5, r_term=10.0, r_outbound=-30.0)
        ctx = StepContext(env, acts, rcfg, target)
        sub = fm.compute_subgrid(env.field, acts, env.grid)
        hx, hy = O.compute_subgrid(env.field, acts.f_max, env.grid)
        assert (sub.half_width_x, sub.half_width_y) == (hx, hy)
        om = O.build_model(env, acts, rcfg, target, hx, hy)
        assert model_digest(fm.build_model(ctx, sub)) == model_digest(om)
        dmc = build_device_model(ctx.device_env(), acts, rcfg, target, sub, lean=False)
        assert model_digest(dmc.to_sparse_model()) == model_digest(om)
        ov, oa, oit, ores, oconv = O.value_iteration(om)
        pv = fm.value_iteration(fm.build_model(ctx, sub))
        assert sha(pv.values) == sha(ov) and sha(pv.actions) == sha(oa)
        assert (pv.iterations_run, pv.residual, pv.converged) == (oit, ores, oconv)


@pytest.mark.parametrize("objective", ["time", "net_energy"])
def test_huge_subgrid_global_histogram(objective):
    """A sub-grid whose per-warp histogram (64 B per slot) exceeds a block's
    shared memory: the build takes the global-histogram kernel (F_GHIST) and
    still matches the reference bit for bit."""
    rng = np.random.default_rng(77)
    nx = ny = 72
    nt, nr, nm = 3, 40, 3
    g = GridSpec(nx=nx, ny=ny, nt=nt, dx=1.0, dt=1.0)
    mask = np.zeros((nt, ny, nx), dtype=bool)
    mask[:, 30:34, 20:26] = True
    env = Environment(grid=g,
                      field=DOVelocityField(mean=rng.uniform(-30.0, 30.0, (nt, ny, nx, 2)),
                                            modes=rng.normal(0, 0.4, (nm, nt, ny, nx, 2)),
                                            coeffs=rng.normal(0, 0.5, (nt, nr, nm))),
                      scalar=ScalarMeanField(g_mean=rng.uniform(0, 2, (nt, ny, nx))),
                      obstacles=ObstacleMask(mask=mask))
    acts = ActionSpace(n_headings=8, n_speeds=1, f_max=1.0)
    rcfg = RewardConfig(objective, c_f=1.0, c_r=0.5, r_term=10.0, r_outbound=-30.0)
    target = (40, 40)
    hx, hy = O.compute_subgrid(env.field, acts.f_max, env.grid)
    assert ((2 * hx + 1) * (2 * hy + 1) + 1) * 64 > 232448   # beyond shared memory
    ctx = StepContext(env, acts, rcfg, target)
    sub = fm.compute_subgrid(env.field, acts, env.grid)
    assert (sub.half_width_x, sub.half_width_y) == (hx, hy)
    om = O.build_model(env, acts, rcfg, target, hx, hy, n_threads=os.cpu_count() or 1)
    assert model_digest(fm.build_model(ctx, sub)) == model_digest(om)
    ov, oa, oit, ores, oconv = O.value_iteration(om)
    assert ores == 0.0
    vals, pol = solve_backward(build_device_model(ctx.device_env(), acts, rcfg, target, sub))
    assert sha(vals.cpu().numpy()) == sha(ov)


@pytest.mark.parametrize("nm", [16, 17, 33, 64, 100, 200])
def test_many_modes(nm):
    """Mode counts past the FP32 filter's register budget (> 16: the plain f64
    scan) and into the hundreds (the build stages them in shared memory with a
    smaller chunk): sub-grid, model and values bit-exact."""
    rng = np.random.default_rng(nm)
    nx, ny, nt, nr = 11, 9, 4, 70
    g = GridSpec(nx=nx, ny=ny, nt=nt, dx=1.0, dt=1.0)
    mask = np.zeros((nt, ny, nx), dtype=bool)
    mask[:, 4, 3:6] = True
    env = Environment(grid=g,
                      field=DOVelocityField(mean=rng.normal(0, 0.6, (nt, ny, nx, 2)),
                                            modes=rng.normal(0, 0.3, (nm, nt, ny, nx, 2)),
                                            coeffs=rng.normal(0, 0.4, (nt, nr, nm))),
                      scalar=ScalarMeanField(g_mean=rng.uniform(0, 2, (nt, ny, nx))),
                      obstacles=ObstacleMask(mask=mask))
    acts = ActionSpace(n_headings=8, n_speeds=1, f_max=1.0)
    from paper_2109_00857_b200.builder import DeviceEnv
    got, want = DeviceEnv.from_host(env).velocity_max(), O.velocity_max(env.field)
    assert np.array(got).tobytes() == np.array(want, dtype=np.float64).tobytes()
    for obj in ("time", "net_energy"):
        rcfg = RewardConfig(obj, c_f=1.0, c_r=0.5, r_term=10.0, r_outbound=-30.0)
        ctx = StepContext(env, acts, rcfg, (8, 7))
        sub = fm.compute_subgrid(env.field, acts, env.grid)
        hx, hy = O.compute_subgrid(env.field, acts.f_max, env.grid)
        assert (sub.half_width_x, sub.half_width_y) == (hx, hy)
        om = O.build_model(env, acts, rcfg, (8, 7), hx, hy)
        assert model_digest(fm.build_model(ctx, sub)) == model_digest(om)
        dmc = build_device_model(ctx.device_env(), acts, rcfg, (8, 7), sub, lean=False)
        assert model_digest(dmc.to_sparse_model()) == model_digest(om)
