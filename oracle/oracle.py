"""ctypes wrapper over ``flowmdp_oracle.c`` -- the CPU parity oracle.

TEST INFRASTRUCTURE ONLY.  Imported by ``tests/``, ``__graft_entry__.smoke``
and ``bench.py`` (cpu_baseline leg and ``--impl reference``), never by the
product package ``paper_2109_00857_b200``.

The C code restates the reference planner's hot path op for op (see the
header of flowmdp_oracle.c for the file:line map).  Inputs are duck-typed:
anything with the reference's attribute names works -- the reference's own
``flowmdp`` dataclasses or this repo's mirrors.  Outputs are plain numpy
containers so the oracle has no dependency on the product package.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "flowmdp_oracle.c")

OBJECTIVE_CODE = {"time": 0, "energy": 1, "net_energy": 2}


def build_lib(force: bool = False) -> str:
    """Compile the oracle (gcc, no FMA contraction).  Idempotent."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["make", "-s", "-C", _HERE, "liboracle.so"],
        )
    return LIB_PATH


class _Problem(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("nt", C.c_int32),
        ("dx", C.c_double), ("dt", C.c_double), ("ox", C.c_double), ("oy", C.c_double),
        ("n_modes", C.c_int32), ("n_real", C.c_int32),
        ("mean", C.c_void_p), ("modes", C.c_void_p), ("coeffs", C.c_void_p),
        ("g", C.c_void_p), ("mask", C.c_void_p),
        ("n_actions", C.c_int32),
        ("avec", C.c_void_p), ("aspeed", C.c_void_p),
        ("objective", C.c_int32),
        ("c_f", C.c_double), ("c_r", C.c_double), ("r_term", C.c_double), ("r_outbound", C.c_double),
        ("target_i", C.c_int32), ("target_j", C.c_int32),
        ("hx", C.c_int32), ("hy", C.c_int32),
        ("rx", C.c_int32), ("ry", C.c_int32),
        ("j0", C.c_int32), ("j1", C.c_int32),
    ]


class _Sparse(C.Structure):
    _fields_ = [
        ("n_g", C.c_int64), ("n_actions", C.c_int32),
        ("off", C.c_void_p), ("rows", C.c_void_p), ("cols", C.c_void_p),
        ("vals", C.c_void_p), ("rewards", C.c_void_p),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_lib()
        L = C.CDLL(LIB_PATH)
        L.or_build.restype = C.c_void_p
        L.or_build.argtypes = [C.POINTER(_Problem), C.c_int]
        L.or_build_range.restype = C.c_void_p
        L.or_build_range.argtypes = [C.POINTER(_Problem), C.c_int, C.c_int, C.c_int]
        L.or_block_nnz.restype = C.c_int64
        L.or_block_nnz.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.or_block_copy.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_rewards_copy.argtypes = [C.c_void_p, C.c_void_p]
        L.or_violation.argtypes = [C.c_void_p, C.c_void_p]
        L.or_model_free.argtypes = [C.c_void_p]
        L.or_velocity_max.argtypes = [C.POINTER(_Problem), C.c_void_p]
        L.or_value_iteration.restype = C.c_double
        L.or_value_iteration.argtypes = [C.POINTER(_Sparse), C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_extract_policy.argtypes = [C.POINTER(_Sparse), C.c_void_p, C.c_void_p]
        L.or_policy_value.argtypes = [C.POINTER(_Sparse), C.c_void_p, C.c_double, C.c_int, C.c_void_p]
        _lib = L
    return _lib


class OracleViolation(Exception):
    """Sub-grid overflow, carrying the reference's message text."""


@dataclass
class OracleModel:
    blocks: list          # [a][t] -> (rows u32, cols u32, vals f64)
    rewards: np.ndarray   # f64 [A * N_g]
    n_states: int
    n_actions: int
    nt: int

    def nnz_total(self) -> int:
        return int(sum(b[0].size for row in self.blocks for b in row))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def velocity_bound(field) -> tuple[float, float]:
    """Triangle-inequality bound (environment.py:404-419), same op order."""
    out = []
    for c in (0, 1):
        per_t = np.abs(field.mean[..., c]).max(axis=(1, 2))
        for m in range(field.modes.shape[0]):
            coeff_max = np.abs(field.coeffs[:, :, m]).max(axis=1)
            mode_max = np.abs(field.modes[m, ..., c]).max(axis=(1, 2))
            per_t = per_t + coeff_max * mode_max
        out.append(float(per_t.max()) if per_t.size else 0.0)
    return out[0], out[1]


def gate_radius(field, f_max: float, grid) -> tuple[int, int]:
    """Obstacle gate radius (model_builder.py:218-223)."""
    bx, by = velocity_bound(field)
    rx = int(math.ceil((bx + f_max) * grid.dt / grid.dx)) + 1
    ry = int(math.ceil((by + f_max) * grid.dt / grid.dx)) + 1
    return rx, ry


def _action_tables(actions):
    """(vectors, speeds) exactly as ActionSpace.vectors/speeds compute them
    (environment.py:220-233): Python-float math on the host."""
    n_h, n_s, f_max = actions.n_headings, actions.n_speeds, actions.f_max
    n_a = n_h * n_s
    vec = np.empty((n_a, 2), dtype=np.float64)
    spd = np.empty(n_a, dtype=np.float64)
    for a in range(n_a):
        h, k = divmod(a, n_s)
        theta = 2.0 * math.pi * h / n_h
        f = f_max * (k + 1) / n_s
        vec[a, 0] = f * math.cos(theta)
        vec[a, 1] = f * math.sin(theta)
        spd[a] = f
    return vec, spd


def _problem(env, actions, rcfg, target, hx=0, hy=0):
    grid, field = env.grid, env.field
    keep = {
        "mean": _f64(field.mean), "modes": _f64(field.modes), "coeffs": _f64(field.coeffs),
        "g": _f64(env.scalar.g_mean),
        "mask": np.ascontiguousarray(env.obstacles.mask, dtype=np.uint8),
    }
    vec, spd = _action_tables(actions)
    keep["avec"], keep["aspeed"] = vec, spd
    rx, ry = gate_radius(field, actions.f_max, grid)
    P = _Problem(
        grid.nx, grid.ny, grid.nt, float(grid.dx), float(grid.dt),
        float(grid.origin[0]), float(grid.origin[1]),
        field.modes.shape[0], field.coeffs.shape[1],
        keep["mean"].ctypes.data, keep["modes"].ctypes.data, keep["coeffs"].ctypes.data,
        keep["g"].ctypes.data, keep["mask"].ctypes.data,
        vec.shape[0], vec.ctypes.data, spd.ctypes.data,
        OBJECTIVE_CODE[rcfg.objective], float(rcfg.c_f), float(rcfg.c_r),
        float(rcfg.r_term), float(rcfg.r_outbound),
        int(target[0]), int(target[1]), int(hx), int(hy), rx, ry, 0, 0,
    )
    return P, keep


def velocity_max(field) -> tuple[float, float]:
    """Exact component-wise max |v| over (t, r, cell) (model_builder.py:392-396)."""
    nt, ny, nx = field.mean.shape[:3]
    keep = [_f64(field.mean), _f64(field.modes), _f64(field.coeffs)]
    P = _Problem()
    P.nx, P.ny, P.nt = nx, ny, nt
    P.n_modes, P.n_real = field.modes.shape[0], field.coeffs.shape[1]
    P.mean, P.modes, P.coeffs = (k.ctypes.data for k in keep)
    out = np.zeros(2)
    lib().or_velocity_max(C.byref(P), out.ctypes.data)
    return float(out[0]), float(out[1])


def compute_subgrid(field, f_max: float, grid, buffer: int = 1) -> tuple[int, int]:
    """model_builder.py:376-399 -> (half_width_x, half_width_y)."""
    vx, vy = velocity_max(field)
    hx = int(math.ceil((vx + f_max) * grid.dt / grid.dx)) + buffer
    hy = int(math.ceil((vy + f_max) * grid.dt / grid.dx)) + buffer
    return hx, hy


def build_model(env, actions, rcfg, target, hx, hy, n_threads: int = 1,
                t_range: tuple[int, int] | None = None,
                j_range: tuple[int, int] | None = None) -> OracleModel:
    """model_builder.py:532-580.  Raises OracleViolation on sub-grid overflow.
    t_range / j_range restrict the build to slabs / source-row strips."""
    P, keep = _problem(env, actions, rcfg, target, hx, hy)
    if j_range is not None:
        P.j0, P.j1 = int(j_range[0]), int(j_range[1])
    L = lib()
    nt = env.grid.nt
    t0, t1 = t_range if t_range is not None else (0, nt)
    h = L.or_build_range(C.byref(P), int(n_threads), int(t0), int(t1))
    try:
        v = np.zeros(5, dtype=np.int32)
        L.or_violation(h, v.ctypes.data)
        if v[0]:
            raise OracleViolation(
                f"displacement ({int(v[3])},{int(v[4])}) at t={int(v[1])}, a={int(v[2])} "
                f"exceeds sub-grid half widths ({hx},{hy})"
            )
        n_a = P.n_actions
        blocks = []
        for a in range(n_a):
            row = []
            for t in range(nt):
                n = L.or_block_nnz(h, a, t)
                rows = np.empty(n, dtype=np.uint32)
                cols = np.empty(n, dtype=np.uint32)
                vals = np.empty(n, dtype=np.float64)
                L.or_block_copy(h, a, t, rows.ctypes.data, cols.ctypes.data, vals.ctypes.data)
                row.append((rows, cols, vals))
            blocks.append(row)
        n_g = env.grid.nx * env.grid.ny * nt
        rewards = np.empty(n_a * n_g, dtype=np.float64)
        L.or_rewards_copy(h, rewards.ctypes.data)
    finally:
        L.or_model_free(h)
    return OracleModel(blocks=blocks, rewards=rewards, n_states=n_g + 1, n_actions=n_a, nt=nt)


def _blocks_of(model):
    """(rows, cols, vals) per block from an OracleModel or a SparseModel-like."""
    out = []
    for row in model.blocks:
        r = []
        for b in row:
            if isinstance(b, tuple):
                r.append(b)
            else:
                r.append((b.rows, b.cols, b.vals))
        out.append(r)
    return out


def _sparse(model):
    blocks = _blocks_of(model)
    n_a = model.n_actions
    off = np.zeros(n_a + 1, dtype=np.int64)
    rows_l, cols_l, vals_l = [], [], []
    for a in range(n_a):
        rs = [b[0] for b in blocks[a]]
        rows_l.append(np.concatenate(rs).astype(np.int64) if rs else np.zeros(0, np.int64))
        cols_l.append(np.concatenate([b[1] for b in blocks[a]]).astype(np.int64) if rs else np.zeros(0, np.int64))
        vals_l.append(np.concatenate([b[2] for b in blocks[a]]).astype(np.float64) if rs else np.zeros(0))
        off[a + 1] = off[a] + rows_l[-1].size
    keep = {
        "off": off,
        "rows": np.ascontiguousarray(np.concatenate(rows_l)),
        "cols": np.ascontiguousarray(np.concatenate(cols_l)),
        "vals": np.ascontiguousarray(np.concatenate(vals_l)),
        "rewards": _f64(model.rewards),
    }
    S = _Sparse(model.n_states - 1, n_a, off.ctypes.data, keep["rows"].ctypes.data,
                keep["cols"].ctypes.data, keep["vals"].ctypes.data, keep["rewards"].ctypes.data)
    return S, keep


def value_iteration(model, epsilon: float = 1e-8, max_iterations: int | None = None):
    """solver.py:75-109 -> (values, actions, iterations_run, residual, converged)."""
    S, keep = _sparse(model)
    max_iter = max_iterations if max_iterations is not None else model.nt + 2
    values = np.empty(model.n_states, dtype=np.float64)
    actions = np.empty(model.n_states - 1, dtype=np.uint16)
    stats = np.zeros(2, dtype=np.int32)
    res = lib().or_value_iteration(C.byref(S), float(epsilon), int(max_iter),
                                   values.ctypes.data, actions.ctypes.data, stats.ctypes.data)
    return values, actions, int(stats[0]), float(res), bool(stats[1])


def extract_policy(model, values):
    S, keep = _sparse(model)
    v = _f64(values)
    out = np.empty(model.n_states - 1, dtype=np.uint16)
    lib().or_extract_policy(C.byref(S), v.ctypes.data, out.ctypes.data)
    return out


def policy_value(model, policy, epsilon: float = 1e-8, max_iterations: int | None = None):
    S, keep = _sparse(model)
    pol = np.ascontiguousarray(policy, dtype=np.uint16)
    max_iter = max_iterations if max_iterations is not None else model.nt + 2
    out = np.empty(model.n_states, dtype=np.float64)
    lib().or_policy_value(C.byref(S), pol.ctypes.data, float(epsilon), int(max_iter), out.ctypes.data)
    return out
