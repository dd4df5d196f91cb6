"""Multi-GPU decomposition logic, exercised on CPU: strip partitioning, halo
planning, and the backward solve with per-layer halo exchange over gloo
(world_size 2 and 3) driven by an oracle layer function.  The GPU run uses
the same code with NCCL and k_solve_layer."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from conftest import make_named_env, make_random_env
from paper_2109_00857_b200.sharding import halo_plan, solve_sharded, strip_bounds


def test_strip_bounds_cover_rows_exactly():
    for ny in (1, 2, 7, 100, 400):
        for world in (1, 2, 3, 4, 8):
            spans = [strip_bounds(ny, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == ny
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and a0 <= a1
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_halo_plan_symmetric_and_sufficient():
    for ny, world, hy in ((100, 8, 5), (13, 4, 6), (10, 3, 1), (9, 8, 3)):
        plans = [halo_plan(ny, world, r, hy) for r in range(world)]
        for r, (sends, recvs) in enumerate(plans):
            j0, j1 = strip_bounds(ny, world, r)
            need = set(range(max(0, j0 - hy), min(ny, j1 + hy))) - set(range(j0, j1))
            got = set()
            for peer, a, b in recvs:
                got |= set(range(a, b))
                # the peer sends exactly this range to me
                assert (r, a, b) in plans[peer][0]
            assert got == need


def _layer_values(model, grid, n_actions, t, j0, j1, values):
    """Reference-order backward layer for rows [j0, j1) (test stand-in for k_solve_layer)."""
    nc = grid.nx * grid.ny
    n_g = nc * grid.nt
    R = model.rewards.reshape(n_actions, n_g)
    for c in range(j0 * grid.nx, j1 * grid.nx):
        s = t * nc + c
        best, best_a = None, 0
        for a in range(n_actions):
            rows, cols, vals = model.blocks[a][t]
            lo, hi = np.searchsorted(rows, [s, s + 1])
            acc = 0.0
            for k in range(lo, hi):
                acc = acc + vals[k] * float(values[cols[k]])
            q = R[a, s] + acc
            if best is None or q > best:
                best, best_a = q, a
        values[s] = best


def _worker(rank, world, port, case, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    env, acts, rcfg, target = case()
    hx, hy = O.compute_subgrid(env.field, acts.f_max, env.grid)
    model = O.build_model(env, acts, rcfg, target, hx, hy)
    g = env.grid
    values = torch.zeros(g.n_states + 1, dtype=torch.float64)
    j0, j1 = strip_bounds(g.ny, world, rank)
    solve_sharded(lambda t: _layer_values(model, g, acts.n_actions, t, j0, j1, values), values,
                  g.nt, g.nx, g.ny, hy)
    mine = np.zeros(g.n_states + 1)
    for t in range(g.nt):
        a, b = t * g.n_cells + j0 * g.nx, t * g.n_cells + j1 * g.nx
        mine[a:b] = values.numpy()[a:b]
    np.save(f"{out_path}.{rank}.npy", mine)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case_random():
    return make_random_env(7004)


def _case_smoke():
    env, acts, rcfg, target, _ = make_named_env("smoke")
    return env, acts, rcfg, target


@pytest.mark.parametrize("case,world", [(_case_random, 2), (_case_smoke, 2), (_case_smoke, 3)])
def test_sharded_backward_solve_gloo(tmp_path, case, world):
    out = str(tmp_path / "v")
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    env, acts, rcfg, target = case()
    hx, hy = O.compute_subgrid(env.field, acts.f_max, env.grid)
    full = O.build_model(env, acts, rcfg, target, hx, hy)
    ref_v, _, _, res, _ = O.value_iteration(full)
    got = sum(np.load(f"{out}.{r}.npy") for r in range(world))
    assert res == 0.0
    assert got.tobytes() == ref_v.tobytes()


def test_weighted_strips_balance_obstacle_cost():
    """Rows near obstacles cost more (per-transition build path): the
    obstacle band's strip gets fewer rows; strips stay contiguous and cover
    every row."""
    from paper_2109_00857_b200.sharding import row_costs, weighted_strips
    env, acts, rcfg, target, _ = make_named_env("desk")
    mask = env.obstacles.mask
    costs = row_costs(mask, 7, 9)
    assert costs.shape == (env.grid.ny,) and (costs >= env.grid.nt * env.grid.nx).all()
    for world in (1, 2, 3, 4, 8):
        b = weighted_strips(costs, world)
        assert b[0][0] == 0 and b[-1][1] == env.grid.ny
        assert all(x1 == y0 for (_, x1), (y0, _) in zip(b, b[1:])) and all(a < c for a, c in b)
        per = [costs[a:c].sum() for a, c in b]
        assert max(per) - min(per) <= costs.max() + 1e-9   # balanced up to one row
    # uniform costs give the equal strips
    assert weighted_strips(np.ones(10), 3) == [strip_bounds(10, 3, r) for r in range(3)] or \
        sorted(c - a for a, c in weighted_strips(np.ones(10), 3)) == [3, 3, 4]


def test_halo_plan_with_uneven_bounds():
    bounds = [(0, 2), (2, 9), (9, 10), (10, 20)]
    for hy in (1, 3, 6):
        plans = [halo_plan(20, 4, r, hy, bounds) for r in range(4)]
        for r, (sends, recvs) in enumerate(plans):
            j0, j1 = bounds[r]
            need = set(range(max(0, j0 - hy), min(20, j1 + hy))) - set(range(j0, j1))
            got = set()
            for peer, a, b in recvs:
                got |= set(range(a, b))
                assert (r, a, b) in plans[peer][0]   # the peer sends exactly these rows
            assert got == need


@pytest.mark.parametrize("nt,n,ratio", [(100, 5, 1.0), (100, 5, 0.7), (100, 6, 0.6), (7, 5, 0.5), (3, 8, 1.0),
                                        (10, 4, 0.3), (200, 5, 1.3)])
def test_slab_groups_partition_descending(nt, n, ratio):
    """The pipelined build's slab groups: a descending partition of [0, nt)
    with every group non-empty; ratio < 1 makes the last groups smaller."""
    from paper_2109_00857_b200.sharding import slab_groups
    gs = slab_groups(nt, n, ratio)
    assert len(gs) == min(n, nt)
    assert gs[0][1] == nt and gs[-1][0] == 0
    assert all(a < b for a, b in gs)
    assert all(gs[k][0] == gs[k + 1][1] for k in range(len(gs) - 1))
    sizes = [b - a for a, b in gs]
    if ratio < 1.0 and nt >= 10 * n:
        assert sizes[-1] < sizes[0]
    if ratio == 1.0:
        assert max(sizes) - min(sizes) <= 1
