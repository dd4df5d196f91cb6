"""Spatial sharding across GPUs.

Source cells are split into y-strips, one per rank.  The build needs no
communication (every (t, cell, action) row depends only on replicated
inputs).  The backward solve has one real exchange per time step: layer t
on strip [j0, j1) reads V_{t+1} on rows [j0 - hy, j1 + hy), so after each
layer every rank sends the rows its neighbours need -- a halo one sub-grid
half-width wide -- with batched point-to-point NCCL (gloo on CPU tests).

The exchange logic is independent of how a layer is computed
(``layer_fn``), which lets the CPU tests drive it with the oracle.
"""

from __future__ import annotations


def strip_bounds(ny: int, world: int, rank: int) -> tuple:
    """Near-equal contiguous row strips [j0, j1)."""
    base, extra = divmod(ny, world)
    j0 = rank * base + min(rank, extra)
    return j0, j0 + base + (1 if rank < extra else 0)


def halo_plan(ny: int, world: int, rank: int, hy: int) -> tuple:
    """(sends, recvs): lists of (peer, r0, r1) row ranges of one layer.

    Rank k needs rows [j0-hy, j1+hy) of V_{t+1}; whatever of that window
    another rank owns is received from it.  Works for strips thinner than
    hy (several peers per side)."""
    sends, recvs = [], []
    mj0, mj1 = strip_bounds(ny, world, rank)
    for peer in range(world):
        if peer == rank:
            continue
        pj0, pj1 = strip_bounds(ny, world, peer)
        # rows of mine the peer needs
        a, b = max(mj0, pj0 - hy), min(mj1, pj1 + hy)
        if a < b:
            sends.append((peer, a, b))
        # rows of the peer I need
        a, b = max(pj0, mj0 - hy), min(pj1, mj1 + hy)
        if a < b:
            recvs.append((peer, a, b))
    return sends, recvs


def host_staged(tensor, group=None) -> bool:
    """True when ``tensor`` lives on a GPU but the group's backend moves host
    memory only (gloo): the exchange then stages through host buffers.  This
    is the test configuration that runs several ranks on one GPU (NCCL
    refuses two ranks on one device); production runs NCCL on device
    buffers."""
    import torch.distributed as dist

    return tensor.is_cuda and dist.get_backend(group) == "gloo"


def all_reduce_max(tensor, group=None) -> None:
    """In-place MAX all-reduce (device buffers under NCCL)."""
    import torch.distributed as dist

    if host_staged(tensor, group):
        h = tensor.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
        tensor.copy_(h)
    else:
        dist.all_reduce(tensor, op=dist.ReduceOp.MAX, group=group)


def all_reduce_sum(tensor, group=None) -> None:
    """In-place SUM all-reduce (device buffers under NCCL)."""
    import torch.distributed as dist

    if host_staged(tensor, group):
        h = tensor.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        tensor.copy_(h)
    else:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)


def exchange_layer(values, t: int, nx: int, ny: int, hy: int, group=None) -> int:
    """Exchange halo rows of layer t of the flat value vector in place.
    Returns the number of bytes this rank sent."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return 0
    sends, recvs = halo_plan(ny, world, rank, hy)
    base = t * nx * ny
    staged = host_staged(values, group)
    ops, landing = [], []
    sent = 0
    for peer, r0, r1 in sends:
        buf = values[base + r0 * nx: base + r1 * nx]
        if staged:
            buf = buf.cpu()
        ops.append(dist.P2POp(dist.isend, buf, peer, group))
        sent += buf.numel() * buf.element_size()
    for peer, r0, r1 in recvs:
        dst = values[base + r0 * nx: base + r1 * nx]
        buf = dst.new_empty(dst.shape, device="cpu") if staged else dst
        if staged:
            landing.append((dst, buf))
        ops.append(dist.P2POp(dist.irecv, buf, peer, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for dst, buf in landing:
        dst.copy_(buf)
    return sent


def solve_sharded(layer_fn, values, nt: int, nx: int, ny: int, hy: int, group=None) -> int:
    """Backward sweep t = nt-1..0: ``layer_fn(t)`` computes this rank's strip
    of layer t into ``values``; the halo of layer t is exchanged before
    layer t-1 reads it.  Returns bytes sent."""
    sent = 0
    for t in range(nt - 1, -1, -1):
        layer_fn(t)
        if t > 0:
            sent += exchange_layer(values, t, nx, ny, hy, group)
    return sent


def device_solve_sharded(dmodel, values, policy, j0: int, j1: int, group=None) -> int:
    """GPU strip solve: k_solve_layer per t + NCCL halo exchange (the
    count -> probability table is built once for all layers)."""
    import ctypes as C

    import torch

    from . import _lib

    g = dmodel.grid
    hy = dmodel.subgrid.half_width_y
    L = _lib.load()
    m = dmodel.fm_model()
    ptab = torch.empty(dmodel.n_real + 1, dtype=torch.float64, device=values.device)
    _lib.check(L.fm_prob_table(int(dmodel.n_real), ptab.data_ptr(), _lib.stream_ptr()), "fm_prob_table")

    def layer(t):
        _lib.check(L.fm_solve_layer_tab(C.byref(m), ptab.data_ptr(), int(t), int(j0), int(j1), values.data_ptr(),
                                        policy.data_ptr(), _lib.stream_ptr()), "fm_solve_layer_tab")

    return solve_sharded(layer, values, g.nt, g.nx, g.ny, hy, group)
