"""The N>1 planner path on real kernels: y-strip builds (k_build), strip
velocity scans + MAX all-reduce (k_vmax), and the strip backward solve
(k_solve_layer) with per-layer halo exchange (sharding.py).

The pool gives one GPU per run and NCCL refuses two ranks on one device, so
the ranks share cuda:0 over gloo (halo and maxima staged through host
memory); everything below the exchange is the production code.  The union
of the strips must equal the oracle's Jacobi values / greedy actions bit for
bit, and every rank must size the same sub-grid as the full scan."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import oracle as O
from conftest import make_named_env, make_random_env

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, case, out_path):
    import torch
    import torch.distributed as dist

    from paper_2109_00857_b200.builder import DeviceEnv, build_device_model, subgrid_from_vmax
    from paper_2109_00857_b200.sharding import device_solve_sharded, strip_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    env, acts, rcfg, target = case()
    g = env.grid
    j0, j1 = strip_bounds(g.ny, world, rank)
    de = DeviceEnv.from_host(env)
    vm = de.velocity_max(j_range=(j0, j1))        # strip scan + all-reduce
    sub = subgrid_from_vmax(vm, acts.f_max, g)
    dm = build_device_model(de, acts, rcfg, target, sub, j_range=(j0, j1))
    values = torch.zeros(g.n_states + 1, dtype=torch.float64, device="cuda")
    policy = torch.zeros(g.n_states, dtype=torch.int16, device="cuda")
    device_solve_sharded(dm, values, policy, j0, j1)
    v, p = values.cpu().numpy(), policy.cpu().numpy().view(np.uint16)
    mine_v, mine_p = np.zeros(g.n_states + 1), np.zeros(g.n_states, dtype=np.uint16)
    for t in range(g.nt):
        a, b = t * g.n_cells + j0 * g.nx, t * g.n_cells + j1 * g.nx
        mine_v[a:b], mine_p[a:b] = v[a:b], p[a:b]
    np.save(f"{out_path}.{rank}.v.npy", mine_v)
    np.save(f"{out_path}.{rank}.p.npy", mine_p)
    np.save(f"{out_path}.{rank}.sub.npy", np.array([sub.half_width_x, sub.half_width_y]))
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


def _case_random_obst():
    return make_random_env(7011)


def _case_smoke():
    env, acts, rcfg, target, _ = make_named_env("smoke")
    return env, acts, rcfg, target


def _case_desk():
    env, acts, rcfg, target, _ = make_named_env("desk")
    return env, acts, rcfg, target


@pytest.mark.parametrize("case,world", [(_case_random, 2), (_case_random_obst, 3), (_case_smoke, 2),
                                        (_case_smoke, 3), (_case_desk, 2), (_case_desk, 4)])
def test_sharded_planner_on_device(tmp_path, case, world):
    import torch.multiprocessing as mp

    out = str(tmp_path / "s")
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    env, acts, rcfg, target = case()
    hx, hy = O.compute_subgrid(env.field, acts.f_max, env.grid)
    for r in range(world):
        assert tuple(np.load(f"{out}.{r}.sub.npy")) == (hx, hy)
    full = O.build_model(env, acts, rcfg, target, hx, hy, n_threads=os.cpu_count() or 1)
    ref_v, ref_a, _, res, _ = O.value_iteration(full)
    g = env.grid
    got_v, got_p = np.zeros(g.n_states + 1), np.zeros(g.n_states, dtype=np.uint16)
    from paper_2109_00857_b200.sharding import strip_bounds
    for r in range(world):   # assemble by copying (a sum would turn -0.0 into +0.0)
        v, p = np.load(f"{out}.{r}.v.npy"), np.load(f"{out}.{r}.p.npy")
        j0, j1 = strip_bounds(g.ny, world, r)
        for t in range(g.nt):
            a, b = t * g.n_cells + j0 * g.nx, t * g.n_cells + j1 * g.nx
            got_v[a:b], got_p[a:b] = v[a:b], p[a:b]
    assert res == 0.0   # finite horizon: Jacobi converges exactly, so the backward sweep must equal it
    assert got_v.tobytes() == ref_v.tobytes()
    assert np.array_equal(got_p, ref_a.astype(np.uint16))


def _planner_worker(rank, world, port, case, out_path, n_groups):
    import torch
    import torch.distributed as dist

    from paper_2109_00857_b200.builder import DeviceEnv
    from paper_2109_00857_b200.sharding import StripPlanner

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    env, acts, rcfg, target = case()
    g = env.grid
    pl = StripPlanner(DeviceEnv.from_host(env), acts, rcfg, target, n_groups=n_groups)
    for _ in range(2):   # the second step reuses the first step's buffers
        dm = pl.step()
    torch.cuda.synchronize()
    assert dm.n_rows == g.nt * (pl.j1 - pl.j0) * g.nx * acts.n_actions   # strip-local row metadata
    v, p = pl.values.cpu().numpy(), pl.policy.cpu().numpy().view(np.uint16)
    np.save(f"{out_path}.{rank}.v.npy", v)
    np.save(f"{out_path}.{rank}.p.npy", p)
    np.save(f"{out_path}.{rank}.b.npy", np.array(pl.bounds))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case,world,n_groups", [(_case_random_obst, 2, 3), (_case_smoke, 3, 4), (_case_desk, 2, 5),
                                                 (_case_desk, 4, 1)])
def test_strip_planner_pipelined(tmp_path, case, world, n_groups):
    """StripPlanner (cost-weighted strips, strip-local models, slab-group
    builds with the per-layer solve + halo exchange on a second stream)
    reproduces the oracle's values and policy bit for bit."""
    import torch.multiprocessing as mp

    out = str(tmp_path / "p")
    mp.spawn(_planner_worker, args=(world, _free_port(), case, out, n_groups), nprocs=world, join=True)
    env, acts, rcfg, target = case()
    hx, hy = O.compute_subgrid(env.field, acts.f_max, env.grid)
    full = O.build_model(env, acts, rcfg, target, hx, hy, n_threads=os.cpu_count() or 1)
    ref_v, ref_a, _, res, _ = O.value_iteration(full)
    g = env.grid
    bounds = [tuple(b) for b in np.load(f"{out}.0.b.npy")]
    assert bounds[0][0] == 0 and bounds[-1][1] == g.ny
    got_v, got_p = np.zeros(g.n_states + 1), np.zeros(g.n_states, dtype=np.uint16)
    for r in range(world):
        v, p = np.load(f"{out}.{r}.v.npy"), np.load(f"{out}.{r}.p.npy")
        assert [tuple(b) for b in np.load(f"{out}.{r}.b.npy")] == bounds   # every rank cut the same strips
        j0, j1 = bounds[r]
        for t in range(g.nt):
            a, b = t * g.n_cells + j0 * g.nx, t * g.n_cells + j1 * g.nx
            got_v[a:b], got_p[a:b] = v[a:b], p[a:b]
    assert res == 0.0
    assert got_v.tobytes() == ref_v.tobytes()
    assert np.array_equal(got_p, ref_a.astype(np.uint16))


def _halo_case_desk():
    env, acts, rcfg, target, _ = make_named_env("desk")
    return env, acts, rcfg, target


@pytest.mark.parametrize("nstrips", [2, 3])
def test_solve_backward_halo_hook(nstrips):
    """fm_solve_backward_halo (the C-ABI strip solve with a halo hook): per
    strip, the hook fills layer t's halo rows -- here from a full-grid
    solve, standing in for the neighbours' NCCL / P2P transfer -- before
    layer t-1 runs; every strip's rows then equal the full solve bit for
    bit, and a hook returning nonzero aborts with FM_BAD_ARG."""
    import ctypes as C

    import torch

    from paper_2109_00857_b200 import _lib
    from paper_2109_00857_b200.builder import DeviceEnv, build_device_model
    from paper_2109_00857_b200.sharding import strip_bounds
    from paper_2109_00857_b200.solver import solve_backward
    import paper_2109_00857_b200 as fm

    env, acts, rcfg, target = _halo_case_desk()
    g = env.grid
    de = DeviceEnv.from_host(env)
    sub = fm.compute_subgrid(env.field, acts, g, device_env=de)
    full_v, full_p = solve_backward(build_device_model(de, acts, rcfg, target, sub))
    hy = sub.half_width_y
    L = _lib.load()
    calls = []
    for k in range(nstrips):
        j0, j1 = strip_bounds(g.ny, nstrips, k)
        dm = build_device_model(de, acts, rcfg, target, sub, j_range=(j0, j1))
        m = dm.fm_model()
        values = torch.zeros(g.n_states + 1, dtype=torch.float64, device="cuda")
        policy = torch.zeros(g.n_states, dtype=torch.int16, device="cuda")

        def hook(user, t, stream, j0=j0, j1=j1, values=values):
            base = t * g.n_cells
            for a, b in ((max(j0 - hy, 0), j0), (j1, min(j1 + hy, g.ny))):
                if a < b:   # the neighbours' rows of V_t, enqueued on the solve stream
                    values[base + a * g.nx:base + b * g.nx].copy_(full_v[base + a * g.nx:base + b * g.nx])
            calls.append(t)
            return 0

        cb = _lib.HALO_FN(hook)
        _lib.check(L.fm_solve_backward_halo(C.byref(m), 0, g.nt, values.data_ptr(), policy.data_ptr(),
                                            C.cast(cb, C.c_void_p), None, _lib.stream_ptr()), "halo solve")
        torch.cuda.synchronize()
        for t in range(g.nt):
            a, b = t * g.n_cells + j0 * g.nx, t * g.n_cells + j1 * g.nx
            assert values[a:b].cpu().numpy().tobytes() == full_v[a:b].cpu().numpy().tobytes(), (k, t)
            assert torch.equal(policy[a:b], full_p[a:b]), (k, t)
    assert calls[:g.nt] == list(range(g.nt - 1, -1, -1))
    # a failing hook aborts the sweep
    bad = _lib.HALO_FN(lambda user, t, stream: 1)
    j0, j1 = strip_bounds(g.ny, nstrips, 0)
    dm = build_device_model(de, acts, rcfg, target, sub, j_range=(j0, j1))
    m = dm.fm_model()
    values = torch.zeros(g.n_states + 1, dtype=torch.float64, device="cuda")
    policy = torch.zeros(g.n_states, dtype=torch.int16, device="cuda")
    st = L.fm_solve_backward_halo(C.byref(m), 0, g.nt, values.data_ptr(), policy.data_ptr(),
                                  C.cast(bad, C.c_void_p), None, _lib.stream_ptr())
    assert st != 0
