"""Parity at the benchmarked configurations (BASELINE.json configs[1..4]).

The bench times C2 (and C3 / C4 as extra lines) at the full 5000 DO
realizations and C5 at 10,000; this file checks exactly those models.  The
whole model stays on the device; three slabs (first, middle, last-before-
horizon) plus the horizon slab are gathered row by row (``rows_coo``) and
compared with the oracle (model_builder.build_model restated in C) bit for
bit: rows, columns, f64 probabilities and rewards of every row and action.
Whole-model properties cover the remaining slabs (every row's counts sum to
N_rv, canonical entry order).

Solve: the planner's backward sweep against the reference-semantics Jacobi
iteration (solver.py:75-109, ``k_jacobi``) on the same model: values within
1e-5 relative (north_star), bit-identical when the Jacobi run ends with
residual 0, and the policy identical except on value ties (both policies
evaluate to the same values within the tolerance).

Reference: model_builder.py:532-580 (build_model), solver.py:75-109."""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

fm = pytest.importorskip("paper_2109_00857_b200")
from paper_2109_00857_b200 import workloads  # noqa: E402
from paper_2109_00857_b200.builder import DeviceEnv, build_device_model, subgrid_from_vmax  # noqa: E402
from paper_2109_00857_b200.solver import solve_backward  # noqa: E402

REL = 1e-5   # north_star: probabilities, rewards and values within 1e-5 relative


def oracle_slab(env, acts, rcfg, target, hx, hy, t, j0, j1, threads=None):
    """Oracle build of slab t, source rows [j0, j1), split into row strips
    run in parallel (ctypes releases the GIL).  Returns per action
    (rows, cols, vals) and the rewards of the slab's cells [A][cells]."""
    threads = threads or os.cpu_count() or 1
    n = max(1, min(threads, j1 - j0))
    cuts = [j0 + (j1 - j0) * k // n for k in range(n + 1)]
    strips = [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if a < b]

    def one(s):
        return O.build_model(env, acts, rcfg, target, hx, hy, n_threads=1, t_range=(t, t + 1), j_range=s)

    with ThreadPoolExecutor(len(strips)) as ex:
        parts = list(ex.map(one, strips))
    g = env.grid
    nc, n_g = g.nx * g.ny, g.nx * g.ny * g.nt
    blocks, rewards = [], []
    for a in range(acts.n_actions):
        blocks.append(tuple(np.concatenate([p.blocks[a][t][k] for p in parts]) for k in range(3)))
        rewards.append(np.concatenate([p.rewards[a * n_g + t * nc + s0 * g.nx: a * n_g + t * nc + s1 * g.nx]
                                       for p, (s0, s1) in zip(parts, strips)]))
    return blocks, rewards


def check_slab_vs_oracle(dm, env, acts, rcfg, target, t, j0, j1):
    sub = dm.subgrid
    blocks, rewards = oracle_slab(env, acts, rcfg, target, sub.half_width_x, sub.half_width_y, t, j0, j1)
    for a in range(acts.n_actions):
        r, c, v, rew = dm.rows_coo(t, a, j0, j1)
        orr, oc, ov = blocks[a]
        assert np.array_equal(r, orr), (t, a, "rows")
        assert np.array_equal(c, oc), (t, a, "cols")
        assert v.tobytes() == ov.tobytes(), (t, a, "vals")
        assert rew.tobytes() == rewards[a].tobytes(), (t, a, "rewards")


def check_row_counts(dm, n_real):
    """Every row's counts sum to N_rv; entries of a row have strictly
    increasing slots (columns ascending, SINK last)."""
    import torch
    g, na = dm.grid, dm.n_actions
    per_layer = g.nx * g.ny * na
    rows_all = dm.row_ptr.numel()
    step = per_layer * max(1, 2_000_000 // per_layer)
    for l0 in range(0, rows_all, step):
        rid = torch.arange(l0, min(rows_all, l0 + step), device=dm.row_ptr.device)
        ptr, cnt = dm.row_ptr[rid], dm.row_nnz[rid].to(torch.int64) & 0xFFFF
        assert bool((cnt > 0).all())
        seg = torch.repeat_interleave(torch.arange(rid.numel(), device=rid.device), cnt)
        idx = torch.repeat_interleave(ptr, cnt) + (torch.arange(int(cnt.sum()), device=rid.device)
                                                   - torch.repeat_interleave(torch.cumsum(cnt, 0) - cnt, cnt))
        ent = dm.entries[idx].to(torch.int64) & 0xFFFFFFFF
        tot = torch.zeros(rid.numel(), dtype=torch.int64, device=rid.device).index_add_(0, seg, ent & 0xFFFF)
        assert bool((tot == n_real).all())
        slot = ent >> 16
        same = seg[1:] == seg[:-1]
        assert bool((slot[1:][same] > slot[:-1][same]).all())


@pytest.mark.parametrize("name", ["paper", "paper_energy", "paper_net_energy"])
def test_bench_config_full_realizations(name):
    """C2 / C3 / C4 exactly as bench.py runs them (5000 realizations)."""
    import torch
    w = workloads.get(name)
    env = w.environment()
    acts, rcfg, target, g = w.actions(), w.reward_config(), w.target, w.grid
    denv = DeviceEnv.from_host(env)
    sub = subgrid_from_vmax(denv.velocity_max(), acts.f_max, g, w.buffer)
    assert (sub.half_width_x, sub.half_width_y) == O.compute_subgrid(env.field, acts.f_max, g)
    dm = build_device_model(denv, acts, rcfg, target, sub)
    for t in (0, g.nt // 2, g.nt - 2, g.nt - 1):
        check_slab_vs_oracle(dm, env, acts, rcfg, target, t, 0, g.ny)
    check_row_counts(dm, w.n_realizations)

    vals, pol = solve_backward(dm)
    vb = vals.cpu().numpy()
    pb = pol.cpu().numpy().view(np.uint16)
    pv = fm.value_iteration(dm)   # reference semantics: Jacobi from 0, epsilon 1e-8
    assert pv.converged
    if pv.residual == 0.0:
        assert vb.tobytes() == pv.values.tobytes()
        assert pb.tobytes() == pv.actions.tobytes()
    else:
        scale = np.maximum(np.abs(pv.values), 1.0)
        assert (np.abs(vb - pv.values) / scale).max() <= REL
        diff = np.nonzero(pb != pv.actions)[0]
        if diff.size:
            # differing actions must be ties: both policies have the same value
            v_ref = fm.policy_value(dm, pv.actions)
            v_ours = fm.policy_value(dm, pb)
            assert (np.abs(v_ref - v_ours) / np.maximum(np.abs(v_ref), 1.0)).max() <= REL
    # the greedy policy at the backward values is the backward policy
    assert np.array_equal(fm.extract_policy(dm, vb), pb)
    del dm
    torch.cuda.empty_cache()


def row_hashes(dm):
    """Per-row digest of the entries (placement-independent: entries of a
    row are in canonical slot order, hashed with their position)."""
    import torch
    cnt = dm.row_nnz.to(torch.int64) & 0xFFFF
    seg = torch.repeat_interleave(torch.arange(cnt.numel(), device=cnt.device), cnt)
    pos = torch.arange(int(cnt.sum()), device=cnt.device) - torch.repeat_interleave(torch.cumsum(cnt, 0) - cnt, cnt)
    idx = torch.repeat_interleave(dm.row_ptr, cnt) + pos
    ent = dm.entries[idx].to(torch.int64) & 0xFFFFFFFF
    key = (ent * 1000003 + pos) * 2654435761 % 4294967291
    return torch.zeros(cnt.numel(), dtype=torch.int64, device=cnt.device).index_add_(0, seg, key)


@pytest.mark.parametrize("name", ["paper", "paper_net_energy"])
def test_build_deterministic_full_realizations(name):
    """Repeated builds of the benchmarked model give the same rows, rewards
    and entries (only the entries' placement may differ): catches scratch
    state leaking between the tasks of a persistent launch (every slab,
    every row -- the oracle comparisons sample four slabs)."""
    import torch
    w = workloads.get(name)
    env = w.environment()
    acts, rcfg, target, g = w.actions(), w.reward_config(), w.target, w.grid
    denv = DeviceEnv.from_host(env)
    sub = subgrid_from_vmax(denv.velocity_max(), acts.f_max, g, w.buffer)
    ref = None
    for _ in range(3):
        dm = build_device_model(denv, acts, rcfg, target, sub)
        dm.check()
        got = (dm.nnz, dm.row_nnz.clone(), dm.reward.clone(), row_hashes(dm))
        if ref is None:
            ref = got
        else:
            assert got[0] == ref[0]
            assert torch.equal(got[1], ref[1]) and torch.equal(got[2], ref[2]) and torch.equal(got[3], ref[3])
        del dm
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_stress_c5_spot_checks():
    """C5 (400x400x200, 32 actions, 10,000 realizations; 1.02e13
    transitions) on one B200: exact sub-grid, full build + backward solve,
    every row's counts sum to N_rv, and slab x row-strip samples bit-exact
    against the oracle (first / middle / last-before-horizon / horizon slab;
    bottom edge, middle and obstacle-band rows)."""
    import torch
    w = workloads.get("stress")
    env = w.environment()
    acts, rcfg, target, g = w.actions(), w.reward_config(), w.target, w.grid
    denv = DeviceEnv.from_host(env)
    sub = subgrid_from_vmax(denv.velocity_max(), acts.f_max, g, w.buffer)
    dm = build_device_model(denv, acts, rcfg, target, sub)
    vals, pol = solve_backward(dm)
    torch.cuda.synchronize()
    check_row_counts(dm, w.n_realizations)
    for t in (0, g.nt // 2, g.nt - 2, g.nt - 1):
        for j0, j1 in ((0, 2), (g.ny // 2 - 1, g.ny // 2 + 1), (g.ny * 11 // 25, g.ny * 11 // 25 + 4)):
            check_slab_vs_oracle(dm, env, acts, rcfg, target, t, j0, j1)
    v = vals.cpu().numpy()
    assert np.isfinite(v).all() and v[-1] == 0.0
    del dm
    torch.cuda.empty_cache()
