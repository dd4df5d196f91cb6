"""Value-iteration solve on the B200: drop-ins for solver.value_iteration /
extract_policy / policy_value (/root/reference/pkg/src/flowmdp/solver.py)
plus the backward-in-time sweep over the compact device model.

Two device paths:

* ``solve_backward(DeviceModel)`` -- the planner's solve.  One Bellman
  layer per time index, t = nt-1 .. 0 (``k_solve_layer``).  The model is a
  DAG in time, so this single pass reaches the fixed point the reference's
  Jacobi iteration converges to; per-row summation order (+0.0 start,
  entry order, R added last) is the reference's, so values and policy are
  bit-identical.
* ``value_iteration(model)`` -- exact reference semantics, including
  ``iterations_run`` / ``residual`` / ``converged`` and a binding
  ``max_iterations``: Jacobi sweeps on a general CSR (``k_jacobi``) with the
  stopping rule evaluated on the device, then the greedy pass.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core_types import PolicyValue, SolverConfig
from .errors import ContractViolation


def _torch():
    import torch
    return torch


# ---------------------------------------------------------------------------
# backward sweep over the compact model
# ---------------------------------------------------------------------------

def solve_backward(dmodel, values=None, policy=None):
    """Values f64 [N_g+1] (SINK = 0) and policy u16-bits [N_g] on the device."""
    torch = _torch()
    g = dmodel.grid
    n_g = g.nt * g.nx * g.ny
    dev = dmodel.reward.device
    if values is None:
        values = torch.zeros(n_g + 1, dtype=torch.float64, device=dev)
    else:
        values[n_g:].zero_()
    if policy is None:
        policy = torch.zeros(n_g, dtype=torch.int16, device=dev)
    m = dmodel.fm_model()
    _lib.check(_lib.load().fm_solve_backward(C.byref(m), 0, g.nt, values.data_ptr(), policy.data_ptr(),
                                             _lib.stream_ptr()), "fm_solve_backward")
    return values, policy


def solve_layer(dmodel, t: int, j0: int, j1: int, values, policy):
    """One backward layer for rows j in [j0, j1) (multi-GPU strips)."""
    m = dmodel.fm_model()
    _lib.check(_lib.load().fm_solve_layer(C.byref(m), int(t), int(j0), int(j1), values.data_ptr(),
                                          policy.data_ptr(), _lib.stream_ptr()), "fm_solve_layer")


# ---------------------------------------------------------------------------
# general CSR (host SparseModel or exported device model)
# ---------------------------------------------------------------------------

@dataclass
class DeviceCsr:
    n_g: int
    n_actions: int
    nt: int
    row_ptr: object   # int64 [A*n_g + 1]
    cols: object      # int32 (u32 bits) [nnz]
    vals: object      # f64 [nnz]
    rewards: object   # f64 [A*n_g]

    def fm_csr(self) -> _lib.FmCsr:
        return _lib.FmCsr(self.n_g, self.n_actions, self.nt, self.row_ptr.data_ptr(), self.cols.data_ptr(),
                          self.vals.data_ptr(), self.rewards.data_ptr())


def _csr_from_triplets(n_g, n_actions, nt, rows, cols, vals, seg_off, rewards, host_arrays=None) -> DeviceCsr:
    torch = _torch()
    L = _lib.load()
    dev = rewards.device
    row_ptr = torch.empty(n_actions * n_g + 1, dtype=torch.int64, device=dev)
    flag = torch.ones(1, dtype=torch.int32, device=dev)
    off = np.ascontiguousarray(seg_off, dtype=np.int64)
    _lib.check(L.fm_csr_row_ptr(rows.data_ptr(), off.ctypes.data, n_actions, n_g, row_ptr.data_ptr(),
                                flag.data_ptr(), _lib.stream_ptr()), "fm_csr_row_ptr")
    if int(flag.item()) != 1:
        # Non-canonical triplet order (never produced by build_model): make
        # each row contiguous with a stable per-action sort so np.bincount's
        # sequential per-row order is preserved, then rebuild row pointers.
        if host_arrays is None:
            host_arrays = (rows.cpu().numpy().view(np.uint32), cols.cpu().numpy().view(np.uint32),
                           vals.cpu().numpy())
        r_h, c_h, v_h = host_arrays
        if r_h.size and int(r_h.max()) >= n_g:
            raise ContractViolation("model rows reference states outside [0, N_g)")
        perm = np.concatenate([off[a] + np.argsort(r_h[off[a]:off[a + 1]], kind="stable")
                               for a in range(n_actions)]) if r_h.size else np.zeros(0, np.int64)
        rows = torch.from_numpy(np.ascontiguousarray(r_h[perm]).view(np.int32)).to(dev)
        cols = torch.from_numpy(np.ascontiguousarray(c_h[perm]).view(np.int32)).to(dev)
        vals = torch.from_numpy(np.ascontiguousarray(v_h[perm])).to(dev)
        _lib.check(L.fm_csr_row_ptr(rows.data_ptr(), off.ctypes.data, n_actions, n_g, row_ptr.data_ptr(),
                                    flag.data_ptr(), _lib.stream_ptr()), "fm_csr_row_ptr")
    return DeviceCsr(n_g, n_actions, nt, row_ptr, cols, vals, rewards)


def csr_from_sparse_model(model, device=None) -> DeviceCsr:
    """Upload a SparseModel's per-action concatenated triplets
    (solver._per_action_triplets, solver.py:55-63)."""
    torch = _torch()
    _lib.load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n_g = model.n_states - 1
    na = model.n_actions
    seg = np.zeros(na + 1, dtype=np.int64)
    parts_r, parts_c, parts_v = [], [], []
    for a in range(na):
        for b in model.blocks[a]:
            parts_r.append(np.asarray(b.rows, dtype=np.uint32))
            parts_c.append(np.asarray(b.cols, dtype=np.uint32))
            parts_v.append(np.asarray(b.vals, dtype=np.float64))
        seg[a + 1] = seg[a] + sum(int(np.asarray(b.rows).size) for b in model.blocks[a])
    r_h = np.concatenate(parts_r) if parts_r else np.zeros(0, np.uint32)
    c_h = np.concatenate(parts_c) if parts_c else np.zeros(0, np.uint32)
    v_h = np.concatenate(parts_v) if parts_v else np.zeros(0)
    if c_h.size and int(c_h.max()) > n_g:
        raise ContractViolation("model cols reference states beyond SINK")
    rewards = np.ascontiguousarray(model.rewards, dtype=np.float64)
    if rewards.size != na * n_g:
        raise ContractViolation("rewards length must equal n_actions * (n_states - 1)")

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    pad = lambda a: a if a.size else np.zeros(1, a.dtype)
    return _csr_from_triplets(n_g, na, model.nt, up(pad(r_h).view(np.int32)), up(pad(c_h).view(np.int32)),
                              up(pad(v_h)), seg, up(rewards), host_arrays=(r_h, c_h, v_h))


def csr_from_device_model(dmodel) -> DeviceCsr:
    """Device-side export of a compact model to the general CSR."""
    block_off, rows, cols, vals, rewards = dmodel.export_device()
    nt, na = dmodel.grid.nt, dmodel.n_actions
    off = block_off.cpu().numpy()
    seg = np.array([off[a * nt] for a in range(na)] + [off[na * nt]], dtype=np.int64)
    n_g = dmodel.n_states - 1
    if rows.numel() == 0:
        torch = _torch()
        rows = torch.zeros(1, dtype=torch.int32, device=rewards.device)
        cols, vals = rows.clone(), torch.zeros(1, dtype=torch.float64, device=rewards.device)
    return _csr_from_triplets(n_g, na, nt, rows, cols, vals, seg, rewards)


def _as_csr(model) -> DeviceCsr:
    if isinstance(model, DeviceCsr):
        return model
    if hasattr(model, "fm_model"):
        return csr_from_device_model(model)
    return csr_from_sparse_model(model)


def _stats(d_stats):
    h = d_stats.cpu().numpy().view(np.uint64)
    return int(h[0]), float(np.array([h[1]], dtype=np.uint64).view(np.float64)[0])


def value_iteration(model, config: SolverConfig = SolverConfig()) -> PolicyValue:
    """Drop-in for solver.value_iteration (solver.py:75-109)."""
    torch = _torch()
    csr = _as_csr(model)
    max_iter = config.max_iterations if config.max_iterations is not None else csr.nt + 2
    dev = csr.rewards.device
    v0 = torch.empty(csr.n_g + 1, dtype=torch.float64, device=dev)
    v1 = torch.empty(csr.n_g + 1, dtype=torch.float64, device=dev)
    st = torch.zeros(2, dtype=torch.int64, device=dev)
    L = _lib.load()
    c = csr.fm_csr()
    _lib.check(L.fm_jacobi(C.byref(c), float(config.epsilon), int(max_iter), v0.data_ptr(), v1.data_ptr(),
                           st.data_ptr(), _lib.stream_ptr()), "fm_jacobi")
    iters, residual = _stats(st)
    v = v0 if iters % 2 == 0 else v1
    act = torch.empty(max(csr.n_g, 1), dtype=torch.int16, device=dev)
    _lib.check(L.fm_greedy(C.byref(c), v.data_ptr(), act.data_ptr(), _lib.stream_ptr()), "fm_greedy")
    values = v.cpu().numpy()
    actions = act.cpu().numpy().view(np.uint16)[: csr.n_g].copy()
    return PolicyValue(values=values, actions=actions, iterations_run=iters, residual=residual,
                       converged=bool(residual < config.epsilon))


def extract_policy(model, values) -> np.ndarray:
    """Drop-in for solver.extract_policy (solver.py:112-119)."""
    torch = _torch()
    values = np.asarray(values, dtype=np.float64)
    if values.shape[0] != model.n_states:
        raise ContractViolation("values length must equal n_states")
    csr = _as_csr(model)
    dev = csr.rewards.device
    v = torch.from_numpy(np.ascontiguousarray(values)).to(dev)
    act = torch.empty(max(csr.n_g, 1), dtype=torch.int16, device=dev)
    _lib.check(_lib.load().fm_greedy(C.byref(csr.fm_csr()), v.data_ptr(), act.data_ptr(), _lib.stream_ptr()),
               "fm_greedy")
    return act.cpu().numpy().view(np.uint16)[: csr.n_g].copy()


def policy_value(model, policy, config: SolverConfig = SolverConfig()) -> np.ndarray:
    """Drop-in for solver.policy_value (solver.py:122-158)."""
    torch = _torch()
    policy = np.asarray(policy)
    if policy.shape[0] != model.n_states - 1:
        raise ContractViolation("policy length must equal n_states - 1")
    csr = _as_csr(model)
    if policy.size and int(policy.max()) >= csr.n_actions:
        raise ContractViolation("policy action index out of range")
    max_iter = config.max_iterations if config.max_iterations is not None else csr.nt + 2
    dev = csr.rewards.device
    pol = torch.from_numpy(np.ascontiguousarray(policy.astype(np.uint16)).view(np.int16)).to(dev)
    v0 = torch.empty(csr.n_g + 1, dtype=torch.float64, device=dev)
    v1 = torch.empty(csr.n_g + 1, dtype=torch.float64, device=dev)
    st = torch.zeros(2, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().fm_policy_value(C.byref(csr.fm_csr()), pol.data_ptr(), float(config.epsilon),
                                           int(max_iter), v0.data_ptr(), v1.data_ptr(), st.data_ptr(),
                                           _lib.stream_ptr()), "fm_policy_value")
    iters, _ = _stats(st)
    return (v0 if iters % 2 == 0 else v1).cpu().numpy()
