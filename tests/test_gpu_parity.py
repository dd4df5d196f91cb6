"""CUDA path vs the CPU oracle, bit for bit, through the drop-in API.

Every comparison is exact (digests over dtype+shape+bytes): transition
counts, CSR indices, probabilities, rewards, values (sign bits included)
and the policy.  The oracle itself is pinned to the reference by
tests/test_oracle_golden.py; where the input digest matches the golden
record, results are also checked against the reference's own digests."""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle as O
from conftest import RANDOM_SEEDS, make_named_env, make_random_env, make_tiny_env, make_zero_flow_env
from golden_util import env_digest, model_digest, sha

pytestmark = pytest.mark.gpu

fm = pytest.importorskip("paper_2109_00857_b200")
from paper_2109_00857_b200 import (  # noqa: E402
    ActionSpace,
    ContractViolation,
    RewardConfig,
    SolverConfig,
    StepContext,
    SubGridSpec,
)
from paper_2109_00857_b200.builder import DeviceEnv, build_device_model  # noqa: E402
from paper_2109_00857_b200.solver import solve_backward  # noqa: E402


def _gpu_case(env, acts, rcfg, target, rec=None):
    """Build + solve on the GPU and on the oracle; assert exact equality."""
    ctx = StepContext(env, acts, rcfg, target)
    sub = fm.compute_subgrid(env.field, acts, env.grid)
    hx, hy = O.compute_subgrid(env.field, acts.f_max, env.grid)
    assert (sub.half_width_x, sub.half_width_y) == (hx, hy)
    gm = fm.build_model(ctx, sub)
    om = O.build_model(env, acts, rcfg, target, hx, hy, n_threads=os.cpu_count() or 1)
    assert gm.nnz_total() == om.nnz_total()
    for a in range(acts.n_actions):
        for t in range(env.grid.nt):
            g, (r, c, v) = gm.blocks[a][t], om.blocks[a][t]
            assert np.array_equal(g.rows, r) and np.array_equal(g.cols, c), (a, t)
            assert sha(g.vals) == sha(v), (a, t)
    assert sha(gm.rewards) == sha(om.rewards)
    assert model_digest(gm) == model_digest(om)

    # drop-in Jacobi value iteration (exact reference semantics)
    pv = fm.value_iteration(gm)
    ov, oa, oit, ores, oconv = O.value_iteration(om)
    assert sha(pv.values) == sha(ov) and sha(pv.actions) == sha(oa)
    assert (pv.iterations_run, pv.residual, pv.converged) == (oit, ores, oconv)

    # planner path: device model + backward sweep
    denv = ctx.device_env()
    dm = build_device_model(denv, acts, rcfg, target, sub)
    vals, pol = solve_backward(dm)
    # the fully checked per-transition path gives the same model
    dmc = build_device_model(denv, acts, rcfg, target, sub, lean=False)
    assert model_digest(dmc.to_sparse_model()) == model_digest(om)
    if ores == 0.0:
        assert sha(vals.cpu().numpy()) == sha(ov)
        assert sha(pol.cpu().numpy().view(np.uint16)) == sha(oa)

    # extract_policy / policy_value drop-ins
    assert np.array_equal(fm.extract_policy(gm, ov), O.extract_policy(om, ov))
    assert sha(fm.policy_value(gm, oa)) == sha(O.policy_value(om, oa))

    if rec is not None and env_digest(env) == rec["input_sha"]:
        assert model_digest(gm) == rec["model_sha"]
        assert sha(pv.values) == rec["solve"]["values_sha"]
        assert sha(pv.actions) == rec["solve"]["actions_sha"]
    return gm, om, pv


@pytest.mark.parametrize("seed", RANDOM_SEEDS)
def test_random_env_parity(golden, seed):
    env, acts, rcfg, target = make_random_env(seed)
    gm, om, _ = _gpu_case(env, acts, rcfg, target, golden["random"][str(seed)])
    for mi in (1, 2, 3):
        pv = fm.value_iteration(gm, SolverConfig(max_iterations=mi))
        v, a, it, res, conv = O.value_iteration(om, max_iterations=mi)
        assert sha(pv.values) == sha(v) and sha(pv.actions) == sha(a)
        assert (pv.iterations_run, pv.residual, pv.converged) == (it, res, conv)


@pytest.mark.parametrize("objective", ["time", "energy", "net_energy"])
def test_tiny_env_parity(golden, objective):
    acts = ActionSpace(n_headings=8, n_speeds=2, f_max=1.0)
    rcfg = RewardConfig(objective=objective, c_f=1.0, c_r=0.8, r_term=50.0, r_outbound=-200.0)
    _gpu_case(make_tiny_env(), acts, rcfg, (4, 4), golden["tiny"][objective])


def test_hand_chain():
    env = make_zero_flow_env(nx=3, ny=1, nt=4, dt=1.0)
    acts = ActionSpace(n_headings=1, n_speeds=1, f_max=1.0)
    rcfg = RewardConfig(objective="time", r_term=10.0, r_outbound=-50.0)
    _, _, pv = _gpu_case(env, acts, rcfg, (2, 0))
    assert pv.values[0] == 8.0 and pv.values[1] == 9.0 and pv.values[env.grid.sink] == 0.0


def test_subgrid_violation_message(golden):
    from paper_2109_00857_b200 import DOVelocityField, Environment, GridSpec, ObstacleMask, ScalarMeanField
    grid = GridSpec(nx=8, ny=4, nt=3, dx=1.0, dt=1.0)
    mean = np.zeros((3, 4, 8, 2))
    mean[..., 0] = 2.0
    env = Environment(grid=grid, field=DOVelocityField(mean, np.zeros((0, 3, 4, 8, 2)), np.zeros((3, 3, 0))),
                      scalar=ScalarMeanField(np.ones((3, 4, 8))),
                      obstacles=ObstacleMask(np.zeros((3, 4, 8), dtype=bool)))
    ctx = StepContext(env, ActionSpace(4, 1, 0.5), RewardConfig("time", r_term=10.0, r_outbound=-100.0), (7, 3))
    with pytest.raises(ContractViolation) as ei:
        fm.build_model(ctx, SubGridSpec(1, 1))
    assert str(ei.value) == golden["violation_message"]


def test_buffer_guard():
    env = make_zero_flow_env()
    with pytest.raises(ContractViolation):
        fm.compute_subgrid(env.field, ActionSpace(4, 1, 1.0), env.grid, buffer=0)


@pytest.mark.parametrize("objective", ["time", "energy", "net_energy"])
def test_smoke_parity(golden, objective):
    env, acts, _, target, start = make_named_env("smoke")
    rcfg = RewardConfig(objective, c_f=1.0, c_r=0.5, r_term=100.0, r_outbound=-300.0)
    rec = golden["named"][f"smoke_{objective}"]
    _, _, pv = _gpu_case(env, acts, rcfg, target, rec)
    assert pv.values[env.grid.state_index(*start, 0)] == rec["v_start"]


@pytest.mark.parametrize("objective", ["time", "energy", "net_energy"])
def test_desk_parity(golden, objective):
    env, acts, _, target, start = make_named_env("desk")
    rcfg = RewardConfig(objective, c_f=1.0, c_r=0.5, r_term=100.0, r_outbound=-300.0)
    rec = golden["named"][f"desk_{objective}"]
    _, _, pv = _gpu_case(env, acts, rcfg, target, rec)
    if env_digest(env) == rec["input_sha"]:
        assert pv.values[env.grid.state_index(*start, 0)] == rec["v_start"]
        assert pv.iterations_run == rec["solve"]["iterations_run"]


def test_strip_and_slab_sharding_union_equals_full():
    """Spatial strips x time slabs built separately produce the same rows.
    A strip's model holds only its own cells' rows (row metadata sized for
    the strip, as each GPU of a multi-GPU build allocates)."""
    env, acts, rcfg, target, _ = make_named_env("smoke")
    denv = DeviceEnv.from_host(env)
    sub = fm.compute_subgrid(env.field, acts, env.grid, device_env=denv)
    full = build_device_model(denv, acts, rcfg, target, sub)
    ny, nt, nx = env.grid.ny, env.grid.nt, env.grid.nx
    fe = full.entries.cpu().numpy()
    covered = 0
    for j0, j1 in ((0, 3), (3, 7), (7, ny)):
        for t0, t1 in ((0, 4), (4, nt)):
            part = build_device_model(denv, acts, rcfg, target, sub, t_range=(t0, t1), j_range=(j0, j1))
            assert part.n_rows == nt * (j1 - j0) * nx * acts.n_actions
            pe = part.entries.cpu().numpy()
            for t in range(t0, t1):
                for a in range(acts.n_actions):
                    _, rp = part.row_ids(t, a, j0, j1)
                    _, rf = full.row_ids(t, a, j0, j1)
                    n_p = part.row_nnz[rp].cpu().numpy()
                    assert np.array_equal(n_p, full.row_nnz[rf].cpu().numpy())
                    assert part.reward[rp].cpu().numpy().tobytes() == full.reward[rf].cpu().numpy().tobytes()
                    for pp, ff, k in zip(part.row_ptr[rp].cpu().numpy(), full.row_ptr[rf].cpu().numpy(), n_p):
                        assert np.array_equal(pe[pp:pp + k], fe[ff:ff + k])
                    covered += rp.numel()
    assert covered == full.n_rows


@pytest.mark.parametrize("name", ["paper", "paper_energy", "paper_net_energy"])
def test_paper_scale_slabs_vs_oracle(name):
    """C2/C3/C4 geometry (100x100, 16 actions; time / energy / net_energy with
    two moving obstacles) with 1000 realizations: every slab on the GPU,
    three slabs (first, middle, horizon) on the oracle."""
    from paper_2109_00857_b200 import workloads
    w = workloads.get(name).with_(grid=workloads.GridSpec(nx=100, ny=100, nt=100, dx=1.0, dt=1.0),
                                     n_realizations=1000)
    env = w.environment()
    acts, rcfg, target = w.actions(), w.reward_config(), w.target
    ctx = StepContext(env, acts, rcfg, target)
    sub = fm.compute_subgrid(env.field, acts, env.grid)
    assert (sub.half_width_x, sub.half_width_y) == O.compute_subgrid(env.field, acts.f_max, env.grid)
    gm = fm.build_model(ctx, sub)
    slabs = (0, 44, 99)
    for t in slabs:
        om = O.build_model(env, acts, rcfg, target, sub.half_width_x, sub.half_width_y,
                           n_threads=os.cpu_count() or 1, t_range=(t, t + 1))
        for a in range(acts.n_actions):
            g = gm.blocks[a][t]
            r, c, v = om.blocks[a][t]
            assert np.array_equal(g.rows, r) and np.array_equal(g.cols, c) and sha(g.vals) == sha(v), (t, a)
        n_g = env.grid.n_states
        nc = env.grid.n_cells
        gr = gm.rewards.reshape(acts.n_actions, n_g)[:, t * nc:(t + 1) * nc]
        orr = om.rewards.reshape(acts.n_actions, n_g)[:, t * nc:(t + 1) * nc]
        assert sha(gr) == sha(orr)
    # size-independent properties over the whole model
    n_r = env.field.n_realizations
    for a in range(acts.n_actions):
        for t in range(env.grid.nt):
            b = gm.blocks[a][t]
            counts = np.rint(b.vals * n_r)
            per_row = np.bincount(b.rows.astype(np.int64) - t * env.grid.n_cells, weights=counts,
                                  minlength=env.grid.n_cells)
            assert (per_row == n_r).all()
            same = np.diff(b.rows.astype(np.int64)) == 0
            assert (np.diff(b.rows.astype(np.int64)) >= 0).all()
            assert (np.diff(b.cols.astype(np.int64))[same] > 0).all()
    # backward sweep vs the reference-semantics Jacobi iteration on the full
    # model.  Jacobi stops once max|dv| < epsilon (solver.py:98), which at
    # this size can happen one sweep before exact convergence; the backward
    # sweep is the exact fixed point, so values agree to within epsilon and
    # the greedy policy at the exact values is the backward policy.
    pv = fm.value_iteration(gm)
    vals, pol = solve_backward(build_device_model(ctx.device_env(), acts, rcfg, target, sub))
    vb = vals.cpu().numpy()
    assert pv.converged
    if pv.residual == 0.0:
        assert sha(vb) == sha(pv.values)
        assert sha(pol.cpu().numpy().view(np.uint16)) == sha(pv.actions)
    else:
        assert np.abs(vb - pv.values).max() <= 1e-6
        assert np.array_equal(fm.extract_policy(gm, vb), pol.cpu().numpy().view(np.uint16))


def test_reference_types_accepted():
    """Objects from another package with the reference's attribute names work."""
    env, acts, rcfg, target = make_random_env(7003)

    class Acts:
        n_headings, n_speeds, f_max = acts.n_headings, acts.n_speeds, acts.f_max

        def vectors(self):
            return acts.vectors()

        def speeds(self):
            return acts.speeds()

        n_actions = acts.n_actions

    ctx = StepContext(env, Acts(), rcfg, target)
    sub = fm.compute_subgrid(env.field, Acts(), env.grid)
    m = fm.build_model(ctx, sub)
    om = O.build_model(env, acts, rcfg, target, sub.half_width_x, sub.half_width_y)
    assert model_digest(m) == model_digest(om)


@pytest.mark.parametrize("case", ["random", "tiny", "smoke", "desk", "paper_1k"])
def test_velocity_max_exact(case):
    """k_vmax (FP32 scan + exact f64 recompute of candidates) equals the
    oracle's exact f64 scan bit for bit (compute_subgrid's vmax)."""
    from paper_2109_00857_b200 import workloads
    envs = []
    if case == "random":
        envs = [make_random_env(s)[0] for s in RANDOM_SEEDS]
    elif case == "tiny":
        envs = [make_tiny_env()]
    elif case == "paper_1k":
        envs = [workloads.get("paper").with_(n_realizations=1000).environment()]
    else:
        envs = [make_named_env(case)[0]]
    for env in envs:
        got = DeviceEnv.from_host(env).velocity_max()
        want = O.velocity_max(env.field)
        assert np.float64(got[0]).tobytes() == np.float64(want[0]).tobytes()
        assert np.float64(got[1]).tobytes() == np.float64(want[1]).tobytes()


@pytest.mark.parametrize("case", ["random", "tiny", "smoke", "desk", "paper_1k", "nan"])
def test_velocity_bounds_and_subgrid(case):
    """fm_velocity_bounds: lo <= the exact max (the oracle's f64 scan) <= hi
    per component, and DeviceEnv.subgrid (bounds when they agree, else the
    exact scan) gives compute_subgrid's half widths (model_builder.py:376-399)
    for buffers 1 and 2; a NaN input makes hi infinite (the exact scan then
    propagates the NaN like numpy)."""
    import math
    import torch
    from paper_2109_00857_b200 import _lib, workloads
    if case == "random":
        cases = [make_random_env(s) for s in RANDOM_SEEDS]
        envs = [(c[0], c[1].f_max) for c in cases]
    elif case == "tiny":
        envs = [(make_tiny_env(), 1.0)]
    elif case == "paper_1k":
        envs = [(workloads.get("paper").with_(n_realizations=1000).environment(), 1.0)]
    elif case == "nan":
        import copy
        env = copy.deepcopy(make_named_env("smoke")[0])
        env.field.coeffs[3, 5, 2] = np.nan
        envs = [(env, 1.0)]
    else:
        envs = [(make_named_env(case)[0], 1.0)]
    for env, f_max in envs:
        de = DeviceEnv.from_host(env)
        g = env.grid
        out = torch.zeros(4, dtype=torch.float64, device="cuda")
        _lib.check(_lib.load().fm_velocity_bounds(de.fm_grid(), de.fm_env(), 0, g.nt, 0, g.ny, out.data_ptr(),
                                                  de._envelope_buf().data_ptr(), _lib.stream_ptr()), "bounds")
        lox, hix, loy, hiy = out.cpu().numpy()
        want = O.velocity_max(env.field)
        if case == "nan":
            assert math.isinf(hix) or math.isinf(hiy)
            continue
        assert lox <= want[0] <= hix and loy <= want[1] <= hiy
        for buf in (1, 2):
            de2 = DeviceEnv.from_host(env)
            sub = de2.subgrid(f_max, buf)
            hw = O.compute_subgrid(env.field, f_max, g, buffer=buf) if buf != 1 else O.compute_subgrid(
                env.field, f_max, g)
            assert (sub.half_width_x, sub.half_width_y) == tuple(hw)


def _decode_envelope(e):
    """int4 order-preserving f32 encodings -> float64 (lo_x, hi_x, lo_y, hi_y)."""
    e = e.astype(np.int64)
    b = np.where(e >= 0, e, e ^ 0x7FFFFFFF).astype(np.uint32)
    return b.view(np.float32).astype(np.float64)


@pytest.mark.parametrize("case,scan", [("desk", "tc"), ("desk", "ffma2"), ("random", "tc"), ("random", "ffma2"),
                                       ("smoke", "tc")])
def test_envelope_contains_exact_velocities(case, scan, monkeypatch):
    """The per-(t, cell) envelope of the bounds scan -- the FFMA2 kernel
    (k_vmax<.., false>, default) or the tensor-core 3xTF32 one (k_vmax_tc,
    FM_TC_SCAN=1) -- contains
    every exact f64 velocity (environment.py:293-297, reference order) and is
    tight (widening well below a cell); its bounds bracket the exact maxima."""
    import torch
    from paper_2109_00857_b200 import _lib
    if scan == "tc":
        monkeypatch.setenv("FM_TC_SCAN", "1")
    else:
        monkeypatch.delenv("FM_TC_SCAN", raising=False)
    envs = [make_random_env(s)[0] for s in RANDOM_SEEDS[:6]] if case == "random" else [make_named_env(case)[0]]
    for env in envs:
        de = DeviceEnv.from_host(env)
        g = env.grid
        out = torch.zeros(4, dtype=torch.float64, device="cuda")
        _lib.check(_lib.load().fm_velocity_bounds(de.fm_grid(), de.fm_env(), 0, g.nt, 0, g.ny, out.data_ptr(),
                                                  de._envelope_buf().data_ptr(), _lib.stream_ptr()), "bounds")
        env_d = _decode_envelope(de._envelope_buf().cpu().numpy())          # [nt][nc][4]
        F = env.field
        nt, nc = g.nt, g.nx * g.ny
        mean = np.asarray(F.mean, np.float64).reshape(nt, nc, 2)
        modes = np.asarray(F.modes, np.float64).reshape(-1, nt, nc, 2)
        coeffs = np.asarray(F.coeffs, np.float64)
        for t in range(nt):
            v = np.broadcast_to(mean[t][None], (coeffs.shape[1], nc, 2)).copy()
            for m in range(modes.shape[0]):   # v = v + c_m * mode_m, ascending m (the reference's order)
                v = v + coeffs[t, :, m][:, None, None] * modes[m, t][None]
            lo, hi = v.min(axis=0), v.max(axis=0)                          # [nc][2]
            e = env_d[t]
            assert np.all(e[:, 0] <= lo[:, 0]) and np.all(hi[:, 0] <= e[:, 1]), (case, t)
            assert np.all(e[:, 2] <= lo[:, 1]) and np.all(hi[:, 1] <= e[:, 3]), (case, t)
            assert np.all(e[:, 1] - e[:, 0] - (hi[:, 0] - lo[:, 0]) <= 1e-3 * (1.0 + np.abs(hi[:, 0]) + np.abs(lo[:, 0])))
            assert np.all(e[:, 3] - e[:, 2] - (hi[:, 1] - lo[:, 1]) <= 1e-3 * (1.0 + np.abs(hi[:, 1]) + np.abs(lo[:, 1])))
        lox, hix, loy, hiy = out.cpu().numpy()
        want = O.velocity_max(env.field)
        assert lox <= want[0] <= hix and loy <= want[1] <= hiy


@pytest.mark.parametrize("name", ["desk", "paper"])
def test_workload_subgrid_hints(name):
    """bench.py's CPU sample uses these pinned sub-grids; the GPU's exact scan must agree."""
    from paper_2109_00857_b200 import workloads
    w = workloads.get(name)
    env = w.environment()
    sub = fm.compute_subgrid(env.field, w.actions(), env.grid)
    assert (sub.half_width_x, sub.half_width_y) == w.subgrid_hint


def test_gate_radius_device_matches_reference_arithmetic():
    """fm_gate_radius (device) == oracle.gate_radius (numpy, the reference's formula)."""
    for seed in RANDOM_SEEDS[:20]:
        env, acts, _, _ = make_random_env(seed)
        de = DeviceEnv.from_host(env)
        got = tuple(int(x) for x in de.gate_radius_device(acts.f_max).cpu().numpy())
        assert got == O.gate_radius(env.field, acts.f_max, env.grid)
        assert de.velocity_bound() == O.velocity_bound(env.field)


def test_planner_deferred_check_and_capacity_retry():
    """plan() queues the solve behind the build; a too-small entry buffer is
    detected by the deferred check, rebuilt and re-solved."""
    env, acts, rcfg, target = make_random_env(7011)
    de = DeviceEnv.from_host(env)
    sub = fm.compute_subgrid(env.field, acts, env.grid, device_env=de)
    dm = build_device_model(de, acts, rcfg, target, sub, capacity_hint=8, defer_check=True)
    v, p = solve_backward(dm)
    assert dm.check() is True
    v, p = solve_backward(dm, v, p)
    hx, hy = sub.half_width_x, sub.half_width_y
    om = O.build_model(env, acts, rcfg, target, hx, hy)
    ov, oa, _, res, _ = O.value_iteration(om)
    if res == 0.0:
        assert v.cpu().numpy().tobytes() == ov.tobytes()
    assert model_digest(dm.to_sparse_model()) == model_digest(om)
    plan = fm.plan(env, acts, rcfg, target)
    if res == 0.0:
        assert plan.values.cpu().numpy().tobytes() == ov.tobytes()


def test_model_buffer_reuse():
    """A build into the buffers of a previous model (reuse=) equals a fresh build."""
    env, acts, rcfg, target = make_random_env(7005)
    de = DeviceEnv.from_host(env)
    sub = fm.compute_subgrid(env.field, acts, env.grid, device_env=de)
    om = O.build_model(env, acts, rcfg, target, sub.half_width_x, sub.half_width_y)
    first = build_device_model(de, acts, rcfg, target, sub)
    other = RewardConfig("net_energy", c_f=1.0, c_r=0.7, r_term=10.0, r_outbound=-60.0)
    second = build_device_model(de, acts, other, target, sub, reuse=first)
    third = build_device_model(de, acts, rcfg, target, sub, reuse=second)
    assert model_digest(third.to_sparse_model()) == model_digest(om)
    part = build_device_model(de, acts, rcfg, target, sub, j_range=(1, 3), reuse=third)
    fresh = build_device_model(de, acts, rcfg, target, sub, j_range=(1, 3))
    import torch
    assert torch.equal(part.row_nnz, fresh.row_nnz) and torch.equal(part.reward, fresh.reward)


@pytest.mark.parametrize("heads", [16, 12])
def test_wide_action_sets_parity(heads):
    """|A| = 32 and 24 (one source cell per warp, C5's action count) on the
    desk world, time and net_energy, every block against the oracle."""
    env, _, _, target, _ = make_named_env("desk")
    acts = ActionSpace(n_headings=heads, n_speeds=2, f_max=1.0)
    for obj in ("time", "net_energy"):
        rcfg = RewardConfig(obj, c_f=1.0, c_r=0.5, r_term=100.0, r_outbound=-300.0)
        _gpu_case(env, acts, rcfg, target)


@pytest.mark.parametrize("heads,speeds", [(3, 1), (5, 1), (3, 2), (7, 1)])
def test_action_counts_not_dividing_a_warp(heads, speeds):
    """|A| = 3, 5, 6, 7: several source cells per warp with a reconstruction
    lane count that does not divide the realization chunk (500 realizations
    span several chunks), time and net_energy, every block vs the oracle."""
    env, _, _, target, _ = make_named_env("desk")
    acts = ActionSpace(n_headings=heads, n_speeds=speeds, f_max=1.0)
    for obj in ("time", "net_energy"):
        rcfg = RewardConfig(obj, c_f=1.0, c_r=0.5, r_term=100.0, r_outbound=-300.0)
        _gpu_case(env, acts, rcfg, target)


def test_velocity_max_row_strips_combine_to_full_scan():
    """fm_velocity_max_rows over y-strips, max-combined (what the ranks'
    all-reduce does), equals the full exact scan bit for bit."""
    for env in (make_named_env("desk")[0], make_random_env(7009)[0]):
        de = DeviceEnv.from_host(env)
        full = de.velocity_max()
        ny = env.grid.ny
        cuts = sorted({0, ny // 3, (2 * ny) // 3, ny})
        parts = []
        for j0, j1 in zip(cuts[:-1], cuts[1:]):
            if j0 < j1:
                de.reset_derived()
                parts.append(de.velocity_max(j_range=(j0, j1)))
        comb = (max(p[0] for p in parts), max(p[1] for p in parts))
        assert np.float64(comb[0]).tobytes() == np.float64(full[0]).tobytes()
        assert np.float64(comb[1]).tobytes() == np.float64(full[1]).tobytes()


@pytest.mark.parametrize("density", [0.04, 0.15])
def test_dense_random_obstacles(density):
    """The desk flow (500 realizations, several chunks) with a random static
    obstacle field: most sources are gated, exact segment tests are frequent
    (the deferred-test queue overflows and drains in several rounds) and
    land-masked slots are everywhere; every objective, every block vs the
    oracle."""
    from paper_2109_00857_b200 import Environment, ObstacleMask
    env0, acts, _, target, _ = make_named_env("desk")
    rng = np.random.default_rng(int(density * 1000))
    mask = rng.random(env0.obstacles.mask.shape) < density
    mask[:, target[1], target[0]] = False
    env = Environment(grid=env0.grid, field=env0.field, scalar=env0.scalar, obstacles=ObstacleMask(mask=mask))
    for obj in ("time", "energy", "net_energy"):
        rcfg = RewardConfig(obj, c_f=1.0, c_r=0.5, r_term=100.0, r_outbound=-300.0)
        _gpu_case(env, acts, rcfg, target)


@pytest.mark.parametrize("slabs", [1, 3, 8, 64])
def test_scanned_upload_matches_full_scan(slabs):
    """DeviceEnv.from_host_scanned (slab-wise H2D with the exact scan of each
    slab overlapping the next copy) uploads the same bytes and yields the
    full scan's maxima bit for bit, for the whole grid and for a row strip."""
    import torch
    for env in (make_named_env("desk")[0], make_random_env(7009)[0], make_named_env("smoke")[0]):
        ref = DeviceEnv.from_host(env)
        full = ref.velocity_max()
        de = DeviceEnv.from_host_scanned(env, slabs=slabs)
        for k in ("mean", "modes", "coeffs", "g", "mask", "sat"):
            assert torch.equal(getattr(de, k), getattr(ref, k)), k
        got = de.velocity_max()
        assert np.float64(got[0]).tobytes() == np.float64(full[0]).tobytes()
        assert np.float64(got[1]).tobytes() == np.float64(full[1]).tobytes()
        ny = env.grid.ny
        j0, j1 = ny // 3, max(ny // 3 + 1, (2 * ny) // 3)
        ref.reset_derived()
        strip = ref.velocity_max(j_range=(j0, j1))
        ds = DeviceEnv.from_host_scanned(env, slabs=slabs, j_range=(j0, j1))
        assert ds.velocity_max(j_range=(j0, j1)) == strip
        pinned = type("E", (), {})()   # pinned torch tensors, the e2e bench's inputs
        pinned.grid = env.grid
        pinned.field = type("F", (), {k: torch.from_numpy(np.ascontiguousarray(getattr(env.field, k))).pin_memory()
                                      for k in ("mean", "modes", "coeffs")})()
        pinned.scalar = type("S", (), {"g_mean": torch.from_numpy(env.scalar.g_mean).pin_memory()})()
        pinned.obstacles = type("O", (), {"mask": torch.from_numpy(env.obstacles.mask.view(np.uint8)).pin_memory()})()
        dp = DeviceEnv.from_host_scanned(pinned, slabs=slabs)
        assert torch.equal(dp.modes, ref.modes) and dp.velocity_max() == full


@pytest.mark.parametrize("case", ["desk", "paper_1k", "two_obstacles_1k", "zero_flow", "random"])
def test_binned_build_equals_per_transition_build(case, monkeypatch):
    """Cells binned per (cell, realization) (k_build's bin path, with the
    scan's per-cell envelope or the in-kernel triangle bound; lean tasks and
    obstacle tasks) give the same model as the per-transition path
    (FM_NO_BINS) and as binning lean tasks only (FM_NO_OBST_BINS), entry for
    entry."""
    import torch
    if case == "desk":
        env, acts, rcfg, target, _ = make_named_env("desk")
    elif case in ("paper_1k", "two_obstacles_1k"):
        from paper_2109_00857_b200 import workloads
        w = workloads.get("paper" if case == "paper_1k" else "paper_net_energy").with_(
            n_realizations=1000, objective="time")
        env, acts, rcfg, target = w.environment(), w.actions(), w.reward_config(), w.target
    elif case == "zero_flow":   # every realization sits exactly on a step: all take the exact path
        env = make_zero_flow_env(nx=12, ny=12, nt=5, n_realizations=64)
        acts, rcfg, target = ActionSpace(8, 2, 1.0), RewardConfig("time", r_term=10.0, r_outbound=-50.0), (9, 9)
    else:
        env, acts, rcfg, target = make_random_env(7005)
    denv = DeviceEnv.from_host(env)
    sub = fm.compute_subgrid(env.field, acts, env.grid, device_env=denv)

    def flat(dm):
        sm = dm.to_sparse_model()
        return model_digest(sm), sm.rewards.tobytes()

    binned = flat(build_device_model(denv, acts, rcfg, target, sub))
    saved = denv._env_rows
    denv._env_rows = None                     # no envelope: triangle bound around the mean
    tri = flat(build_device_model(denv, acts, rcfg, target, sub))
    denv._env_rows = saved
    monkeypatch.setenv("FM_NO_OBST_BINS", "1")
    lean_only = flat(build_device_model(denv, acts, rcfg, target, sub))
    monkeypatch.setenv("FM_NO_BINS", "1")
    ref = flat(build_device_model(denv, acts, rcfg, target, sub))
    assert binned == ref and tri == ref and lean_only == ref
    torch.cuda.synchronize()


@pytest.mark.parametrize("case", ["smoke", "desk", "two_obstacles_1k"])
def test_reward_sum_counts_net_energy(case, monkeypatch):
    """reward_sum="counts" (fm_build_args.reward_mode 1): net-energy rows
    take the binned build; every COO block (rows, cols, f64 probabilities)
    stays bit-identical to the oracle's and every reward agrees with the
    reference's sequential sum (model_builder.py:457-458) within 1e-12
    relative (north_star allows 1e-5)."""
    from paper_2109_00857_b200 import workloads
    if case == "two_obstacles_1k":
        w = workloads.get("paper_net_energy").with_(n_realizations=1000)
        env, acts, rcfg, target = w.environment(), w.actions(), w.reward_config(), w.target
    else:
        env, acts, rcfg, target, _ = make_named_env(case)
        rcfg = type(rcfg)(objective="net_energy", c_f=rcfg.c_f, c_r=rcfg.c_r, r_term=rcfg.r_term,
                          r_outbound=rcfg.r_outbound)
    denv = DeviceEnv.from_host(env)
    sub = fm.compute_subgrid(env.field, acts, env.grid, device_env=denv)
    om = O.build_model(env, acts, rcfg, target, sub.half_width_x, sub.half_width_y)
    sm = build_device_model(denv, acts, rcfg, target, sub, reward_sum="counts").to_sparse_model()
    for a in range(acts.n_actions):
        for t in range(env.grid.nt):
            r, c, v = om.blocks[a][t]
            b = sm.blocks[a][t]
            assert np.array_equal(b.rows, r) and np.array_equal(b.cols, c) and b.vals.tobytes() == v.tobytes()
    rel = np.abs(sm.rewards - om.rewards) / np.maximum(np.abs(om.rewards), 1.0)
    assert rel.max() <= 1e-12
    seq = build_device_model(denv, acts, rcfg, target, sub).to_sparse_model()
    assert seq.rewards.tobytes() == om.rewards.tobytes()   # the default stays bit-exact
    # the binned rows sum only their slot range; the per-transition path
    # sums every slot -- same slot order, so the same bits
    monkeypatch.setenv("FM_NO_BINS", "1")
    pt = build_device_model(denv, acts, rcfg, target, sub, reward_sum="counts").to_sparse_model()
    assert pt.rewards.tobytes() == sm.rewards.tobytes()
