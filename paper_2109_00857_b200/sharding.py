"""Spatial sharding across GPUs.

Source cells are split into y-strips, one per rank.  The build needs no
communication (every (t, cell, action) row depends only on replicated
inputs).  The backward solve has one real exchange per time step: layer t
on strip [j0, j1) reads V_{t+1} on rows [j0 - hy, j1 + hy), so after each
layer every rank sends the rows its neighbours need -- a halo one sub-grid
half-width wide -- with batched point-to-point NCCL (gloo on CPU tests).

Strips are cut by cost, not by row count: cells near an obstacle take the
per-transition path of k_build (the exact segment tests), several times the
cost of the binned lean cells, so a strip through the obstacle band gets
fewer rows (``row_costs`` / ``weighted_strips``).

``StripPlanner`` is the multi-GPU planner step: per-strip exact scan + MAX
all-reduce, strip-local model (row metadata for the strip's cells only),
the build launched in descending slab groups, and the per-layer solve + halo
exchange of a group running on a second stream while the next groups build
-- so the halo latency chain hides under the build except for the last
group.  The reference's only parallelism is its fork pool over time slabs
(model_builder.py:548-566).

The exchange logic is independent of how a layer is computed
(``layer_fn``), which lets the CPU tests drive it with the oracle.
"""

from __future__ import annotations

import numpy as np


def strip_bounds(ny: int, world: int, rank: int) -> tuple:
    """Near-equal contiguous row strips [j0, j1)."""
    base, extra = divmod(ny, world)
    j0 = rank * base + min(rank, extra)
    return j0, j0 + base + (1 if rank < extra else 0)


def equal_strips(ny: int, world: int) -> list:
    return [strip_bounds(ny, world, r) for r in range(world)]


def row_costs(mask: np.ndarray, rx: int, ry: int, w_obst: float = 8.0) -> np.ndarray:
    """Estimated build cost per source row j (summed over layers and
    columns): 1 per lean cell, ``w_obst`` per cell whose obstacle gate --
    the box of half-widths (rx, ry) -- touches the mask at t or t + 1 (those
    cells take the per-transition path with exact segment tests; the
    horizon layer costs 1).  Deterministic: every rank computes the same
    strips from the same inputs."""
    m = np.asarray(mask).astype(bool)
    nt, ny, nx = m.shape
    near = np.zeros((nt, ny, nx), dtype=bool)
    if nt > 1:
        both = m[:-1] | m[1:]
        sat = np.zeros((nt - 1, ny + 1, nx + 1), dtype=np.int64)
        sat[:, 1:, 1:] = both.cumsum(1).cumsum(2)
        j = np.arange(ny)
        i = np.arange(nx)
        j0, j1 = np.clip(j - ry, 0, ny), np.clip(j + ry + 1, 0, ny)
        i0, i1 = np.clip(i - rx, 0, nx), np.clip(i + rx + 1, 0, nx)
        box = (sat[:, j1][:, :, i1] - sat[:, j0][:, :, i1] - sat[:, j1][:, :, i0] + sat[:, j0][:, :, i0])
        near[:-1] = box > 0
    return (1.0 + (w_obst - 1.0) * near).sum(axis=(0, 2))


def weighted_strips(costs: np.ndarray, world: int) -> list:
    """Contiguous strips [j0, j1) with near-equal summed cost (every strip
    gets at least one row)."""
    ny = len(costs)
    if world > ny:
        raise ValueError(f"{world} ranks for {ny} rows")
    cum = np.concatenate([[0.0], np.cumsum(costs)])
    cuts = [0]
    for r in range(1, world):
        target = cum[-1] * r / world
        j = int(np.searchsorted(cum, target))
        if j > 0 and abs(cum[j - 1] - target) <= abs(cum[j] - target):
            j -= 1
        j = max(j, cuts[-1] + 1)
        j = min(j, ny - (world - r))
        cuts.append(j)
    cuts.append(ny)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def halo_plan(ny: int, world: int, rank: int, hy: int, bounds: list | None = None) -> tuple:
    """(sends, recvs): lists of (peer, r0, r1) row ranges of one layer.

    Rank k needs rows [j0-hy, j1+hy) of V_{t+1}; whatever of that window
    another rank owns is received from it.  Works for strips thinner than
    hy (several peers per side).  ``bounds``: every rank's strip (default:
    equal strips)."""
    bounds = bounds if bounds is not None else equal_strips(ny, world)
    sends, recvs = [], []
    mj0, mj1 = bounds[rank]
    for peer in range(world):
        if peer == rank:
            continue
        pj0, pj1 = bounds[peer]
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


def exchange_layer(values, t: int, nx: int, ny: int, hy: int, group=None, bounds: list | None = None) -> int:
    """Exchange halo rows of layer t of the flat value vector in place
    (on the current stream).  Returns the number of bytes this rank sent."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return 0   # one process: nothing to exchange
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return 0
    sends, recvs = halo_plan(ny, world, rank, hy, bounds)
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


def solve_sharded(layer_fn, values, nt: int, nx: int, ny: int, hy: int, group=None, bounds: list | None = None,
                  t_range: tuple | None = None) -> int:
    """Backward sweep t = t1-1..t0: ``layer_fn(t)`` computes this rank's
    strip of layer t into ``values``; the halo of layer t is exchanged before
    layer t-1 reads it.  Returns bytes sent."""
    t0, t1 = t_range if t_range is not None else (0, nt)
    sent = 0
    for t in range(t1 - 1, t0 - 1, -1):
        layer_fn(t)
        if t > 0:
            sent += exchange_layer(values, t, nx, ny, hy, group, bounds)
    return sent


def _solve_layer_fn(dmodel, values, policy, j0: int, j1: int):
    """k_solve_layer over the strip, the count -> probability table built once."""
    import ctypes as C

    import torch

    from . import _lib
    L = _lib.load()
    m = dmodel.fm_model()
    ptab = torch.empty(dmodel.n_real + 1, dtype=torch.float64, device=values.device)
    _lib.check(L.fm_prob_table(int(dmodel.n_real), ptab.data_ptr(), _lib.stream_ptr()), "fm_prob_table")

    def layer(t):
        _lib.check(L.fm_solve_layer_tab(C.byref(m), ptab.data_ptr(), int(t), int(j0), int(j1), values.data_ptr(),
                                        policy.data_ptr(), _lib.stream_ptr()), "fm_solve_layer_tab")

    layer.keep = (m, ptab)
    return layer


def device_solve_sharded(dmodel, values, policy, j0: int, j1: int, group=None, bounds: list | None = None) -> int:
    """GPU strip solve: k_solve_layer per t + NCCL halo exchange."""
    g = dmodel.grid
    layer = _solve_layer_fn(dmodel, values, policy, j0, j1)
    return solve_sharded(layer, values, g.nt, g.nx, g.ny, dmodel.subgrid.half_width_y, group, bounds)


def slab_groups(nt: int, n_groups: int, ratio: float = 1.0) -> list:
    """Descending slab groups [(t0, t1), ...] covering [0, nt), the last
    layers first (the backward solve's order).  Group k (in launch order)
    gets a share of the slabs proportional to ratio**k: with ratio < 1 the
    groups shrink toward t = 0, so the work left after the last group's
    build -- its layers' solve and its share of the model's device-to-host
    copy -- is small.  Every group holds at least one slab."""
    n = max(1, min(n_groups, nt))
    if not ratio > 0.0:
        raise ValueError("ratio must be > 0")
    w = [ratio ** k for k in range(n)]   # launch order: highest t first
    tot = sum(w)
    sizes, acc, done = [], 0.0, 0
    for k in range(n):
        acc += w[k]
        end = nt if k == n - 1 else int(round(nt * acc / tot))
        end = max(end, done + 1)             # >= 1 slab per group
        end = min(end, nt - (n - 1 - k))     # leave >= 1 slab for each later group
        sizes.append(end - done)
        done = end
    out, hi = [], nt
    for sz in sizes:
        out.append((hi - sz, hi))
        hi -= sz
    return out


class StripPlanner:
    """The multi-GPU planner step (one process per GPU; also runs with one).

    Per step: exact sub-grid scan of this rank's strip + MAX all-reduce
    (every rank gets the global sub-grid and the same proofs); the strip's
    build, launched in descending slab groups; on a second stream, per
    group: wait for its build, then per layer t (descending) k_solve_layer
    on the strip and the halo exchange of layer t.  The deferred build check
    is collective: if any rank had to rebuild (capacity) all ranks solve
    again, and a sub-grid violation on any rank raises on every rank."""

    def __init__(self, denv, actions, rcfg, target, buffer: int = 1, group=None, n_groups: int = 6,
                 reserve_sms: int = 2, w_obst: float = 8.0, bounds: list | None = None,
                 reward_sum: str = "sequential", group_ratio: float = 0.6):
        import torch
        import torch.distributed as dist

        self.denv, self.actions, self.rcfg, self.target = denv, actions, rcfg, target
        self.buffer, self.group = buffer, group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        g = denv.grid
        if bounds is None:
            rxy = denv.gate_radius_device(float(actions.f_max)).cpu().numpy()
            bounds = weighted_strips(row_costs(denv.mask.cpu().numpy(), int(rxy[0]), int(rxy[1]), w_obst),
                                     self.world)
        self.bounds = bounds
        self.j0, self.j1 = bounds[self.rank]
        self.n_groups, self.reserve_sms = n_groups, reserve_sms
        self.group_ratio = group_ratio
        self.reward_sum = reward_sum   # build_device_model: "sequential" (bit-exact) or "counts"
        dev = denv.mean.device
        self.values = torch.zeros(g.nt * g.nx * g.ny + 1, dtype=torch.float64, device=dev)
        self.policy = torch.zeros(g.nt * g.nx * g.ny, dtype=torch.int16, device=dev)
        self.solve_stream = torch.cuda.Stream(device=dev, priority=-1)
        self.dm = None
        self.events = {}

    def _solve(self, dm, pipelined: bool, after=None):
        import torch
        g = dm.grid
        hy = dm.subgrid.half_width_y
        main = torch.cuda.current_stream()
        ss = self.solve_stream if pipelined else main
        if pipelined:
            # the main-stream work before this step's build (``after``: an
            # event recorded ahead of the build launches -- waiting on the
            # main stream itself here would wait for the whole build and
            # serialise the solve behind it); each group's layers then wait
            # for that group's build event below
            if after is not None:
                ss.wait_event(after)
            else:
                ss.wait_stream(main)
        with torch.cuda.stream(ss):
            self.values[-1:].zero_()
            layer = _solve_layer_fn(dm, self.values, self.policy, self.j0, self.j1)
            groups = dm.group_events if pipelined and dm.group_events else [((0, g.nt), None)]
            for (t0, t1), ev in groups:
                if ev is not None:
                    ss.wait_event(ev)
                solve_sharded(layer, self.values, g.nt, g.nx, g.ny, hy, self.group, self.bounds, (t0, t1))
        if pipelined:
            main.wait_stream(ss)

    def step(self, scanned: bool = False, sink: dict | None = None, sink_stream=None):
        """One planner step; returns the strip's DeviceModel (values /
        policy in ``self.values`` / ``self.policy``).  With ``sink`` (pinned
        host buffers, DeviceModel.host_buffers) the compact model streams to
        the host on ``sink_stream`` group by group while the build runs;
        ``self.sink_bytes`` = the bytes copied."""
        import torch

        from .builder import build_device_model
        de, g = self.denv, self.denv.grid
        if not scanned:
            de.reset_derived()
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        self.events = {"start": ev(), "scanned": ev(), "built": ev(), "solved": ev()}
        self.events["start"].record()
        if self.world > 1:
            sub = de.subgrid(self.actions.f_max, self.buffer, j_range=(self.j0, self.j1), group=self.group)
        else:
            sub = de.subgrid(self.actions.f_max, self.buffer)
        self.events["scanned"].record()
        dm = build_device_model(de, self.actions, self.rcfg, self.target, sub, j_range=(self.j0, self.j1),
                                defer_check=True, reuse=self.dm, t_groups=slab_groups(g.nt, self.n_groups, self.group_ratio),
                                reserve_sms=self.reserve_sms, reward_sum=self.reward_sum)
        self.dm = dm
        self.events["built"].record()
        self._solve(dm, pipelined=True, after=self.events["scanned"])
        self.events["solved"].record()
        self.sink_bytes = 0
        if sink is not None:
            self.sink_bytes = dm.stream_to_host(sink, sink_stream)
        if self._finish(dm) and sink is not None:   # rebuilt (capacity): copy the final model again
            sink_stream.wait_stream(torch.cuda.current_stream())
            self.sink_bytes = dm.copy_to_host(sink, sink_stream)
        return dm

    def _finish(self, dm):
        """Deferred build check, collective-safe: every rank learns whether
        any rank rebuilt (capacity) or failed (sub-grid violation)."""
        import torch
        err, rebuilt = None, False
        try:
            rebuilt = dm.check()
        except Exception as exc:   # re-raised after the ranks agree
            err = exc
        if self.world > 1:
            flag = torch.tensor([float(rebuilt), float(err is not None)], dtype=torch.float64,
                                device=self.values.device)
            all_reduce_max(flag, self.group)
            if flag[1].item() and err is None:
                raise RuntimeError("k_build check failed on another rank")
            rebuilt = bool(flag[0].item())
        if err is not None:
            raise err
        if rebuilt:   # capacity miss somewhere: the model was rebuilt, solve again (all ranks)
            self._solve(dm, pipelined=False)
        return rebuilt
