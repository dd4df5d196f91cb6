"""Value types of the drop-in boundary.

Field names, shapes, index conventions and validation errors follow the
reference API so that code written against ``flowmdp`` runs unchanged:

    GridSpec / DOVelocityField / ScalarMeanField / ObstacleMask /
    ActionSpace / Environment      environment.py:30-253
    RewardConfig / SubGridSpec / CooBlock / SparseModel / StepContext
                                   model_builder.py:54-259
    SolverConfig / PolicyValue     solver.py:25-52

Every function of this package is duck-typed: the reference's own
dataclasses can be passed wherever these are expected.  Host-side
derived constants (action vectors, cell centres, reward bases) are
computed here with Python floats in the reference's operation order; the
per-transition arithmetic runs on the GPU (csrc/flowmdp_b200.cu).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ContractViolation

OUTSIDE = -1
OBJECTIVES = ("time", "energy", "net_energy")
OBJECTIVE_CODE = {"time": 0, "energy": 1, "net_energy": 2}


def _require(cond: bool, msg: str) -> None:
    if not cond:
        raise ContractViolation(msg)


# ---------------------------------------------------------------------------
# environment
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class GridSpec:
    """Square cells, half-open; state s = t*N_c + j*nx + i, SINK = N_g."""

    nx: int
    ny: int
    nt: int
    dx: float
    dt: float
    origin: tuple = (0.0, 0.0)

    def __post_init__(self):
        _require(min(self.nx, self.ny, self.nt) >= 1, "grid dimensions must be >= 1")
        _require(self.dx > 0 and self.dt > 0, "dx and dt must be > 0")

    n_cells = property(lambda self: self.nx * self.ny)
    n_states = property(lambda self: self.nx * self.ny * self.nt)
    sink = property(lambda self: self.nx * self.ny * self.nt)

    def state_index(self, i: int, j: int, t: int) -> int:
        _require(0 <= i < self.nx and 0 <= j < self.ny and 0 <= t < self.nt,
                 f"cell ({i},{j},{t}) outside grid")
        return (t * self.ny + j) * self.nx + i

    def split_index(self, s: int) -> tuple:
        _require(0 <= s < self.n_states, f"state index {s} out of range")
        t, rem = divmod(s, self.n_cells)
        j, i = divmod(rem, self.nx)
        return i, j, t

    def cell_center(self, i: int, j: int) -> np.ndarray:
        return np.array([self.origin[0] + (i + 0.5) * self.dx,
                         self.origin[1] + (j + 0.5) * self.dx])

    def center_of(self, s: int) -> np.ndarray:
        i, j, _ = self.split_index(s)
        return self.cell_center(i, j)

    def cell_centers(self) -> np.ndarray:
        xs = self.origin[0] + (np.arange(self.nx, dtype=np.float64) + 0.5) * self.dx
        ys = self.origin[1] + (np.arange(self.ny, dtype=np.float64) + 0.5) * self.dx
        out = np.empty((self.ny, self.nx, 2))
        out[..., 0] = xs[None, :]
        out[..., 1] = ys[:, None]
        return out.reshape(-1, 2)


def _finite(name: str, arr) -> None:
    _require(bool(np.all(np.isfinite(arr))), f"non-finite values in {name}")


@dataclass(frozen=True)
class DOVelocityField:
    """v(t, r, cell) = mean[t, cell] + sum_m coeffs[t, r, m] * modes[m, t, cell]."""

    mean: np.ndarray     # [nt][ny][nx][2]
    modes: np.ndarray    # [n_modes][nt][ny][nx][2]
    coeffs: np.ndarray   # [nt][n_realizations][n_modes]

    def __post_init__(self):
        nt, ny, nx, two = self.mean.shape
        _require(two == 2, "mean must have 2 velocity components")
        _require(tuple(self.modes.shape[1:]) == (nt, ny, nx, 2),
                 f"modes shape {self.modes.shape} inconsistent with mean {self.mean.shape}")
        _require(self.coeffs.shape[0] == nt and self.coeffs.shape[2] == self.modes.shape[0],
                 f"coeffs shape {self.coeffs.shape} inconsistent with nt={nt}, "
                 f"n_modes={self.modes.shape[0]}")
        for name in ("mean", "modes", "coeffs"):
            _finite(name, getattr(self, name))

    n_modes = property(lambda self: self.modes.shape[0])
    n_realizations = property(lambda self: self.coeffs.shape[1])
    nt = property(lambda self: self.mean.shape[0])
    n_cells = property(lambda self: self.mean.shape[1] * self.mean.shape[2])


@dataclass(frozen=True)
class ScalarMeanField:
    g_mean: np.ndarray   # [nt][ny][nx]

    def __post_init__(self):
        _require(self.g_mean.ndim == 3, "g_mean must be indexed [t][y][x]")
        _finite("g_mean", self.g_mean)


@dataclass(frozen=True)
class ObstacleMask:
    mask: np.ndarray     # bool [nt][ny][nx]

    def __post_init__(self):
        _require(self.mask.ndim == 3 and self.mask.dtype == np.bool_,
                 "mask must be a boolean [t][y][x] array")


@dataclass(frozen=True)
class ActionSpace:
    """a = h*n_speeds + k; vector F*(cos th, sin th), th = 2*pi*h/N_h,
    F = f_max*(k+1)/n_speeds (environment.py:187-233)."""

    n_headings: int
    n_speeds: int
    f_max: float

    def __post_init__(self):
        _require(self.n_headings >= 1 and self.n_speeds >= 1, "need at least one heading and one speed")
        _require(self.f_max > 0, "f_max must be > 0")

    n_actions = property(lambda self: self.n_headings * self.n_speeds)

    def heading_index(self, a: int) -> int:
        return a // self.n_speeds

    def speed_index(self, a: int) -> int:
        return a % self.n_speeds

    def speed(self, a: int) -> float:
        return self.f_max * (a % self.n_speeds + 1) / self.n_speeds

    def vectors(self) -> np.ndarray:
        out = np.empty((self.n_actions, 2))
        for a in range(self.n_actions):
            theta = 2.0 * math.pi * (a // self.n_speeds) / self.n_headings
            f = self.speed(a)
            out[a] = (f * math.cos(theta), f * math.sin(theta))
        return out

    def speeds(self) -> np.ndarray:
        return np.array([self.speed(a) for a in range(self.n_actions)])


@dataclass(frozen=True)
class Environment:
    grid: GridSpec
    field: DOVelocityField
    scalar: ScalarMeanField
    obstacles: ObstacleMask

    def __post_init__(self):
        shape = (self.grid.nt, self.grid.ny, self.grid.nx)
        _require(tuple(self.field.mean.shape[:3]) == shape, "velocity field dims do not match grid")
        _require(tuple(self.scalar.g_mean.shape) == shape, "scalar field dims do not match grid")
        _require(tuple(self.obstacles.mask.shape) == shape, "obstacle mask dims do not match grid")


def storage_footprint(field) -> tuple:
    """(reduced, full) scalar counts (environment.py:385-401)."""
    nt, ny, nx = field.mean.shape[:3]
    n_g, n_m, n_rv = nt * ny * nx, field.modes.shape[0], field.coeffs.shape[1]
    return 2 * (1 + n_m) * n_g + n_m * n_rv * nt, 2 * n_g * n_rv


# ---------------------------------------------------------------------------
# model build
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class RewardConfig:
    objective: str
    c_f: float = 1.0
    c_r: float = 1.0
    r_term: float = 100.0
    r_outbound: float = -1000.0

    def __post_init__(self):
        _require(self.objective in OBJECTIVES,
                 f"objective must be one of {OBJECTIVES}, got {self.objective!r}")
        _require(self.r_term > 0, "r_term must be > 0")
        _require(self.r_outbound < 0, "r_outbound must be < 0")


@dataclass(frozen=True)
class SubGridSpec:
    """Displacement window; slot = (dj+hy)(2hx+1) + (di+hx), OUT slot = n_slots."""

    half_width_x: int
    half_width_y: int

    def __post_init__(self):
        _require(self.half_width_x >= 0 and self.half_width_y >= 0, "sub-grid half widths must be >= 0")

    @property
    def n_slots(self) -> int:
        return (2 * self.half_width_x + 1) * (2 * self.half_width_y + 1)

    @property
    def out_slot(self) -> int:
        return self.n_slots

    def slot_of(self, di: int, dj: int) -> int:
        hx, hy = self.half_width_x, self.half_width_y
        _require(abs(di) <= hx and abs(dj) <= hy, f"displacement ({di},{dj}) outside sub-grid")
        return (dj + hy) * (2 * hx + 1) + di + hx


@dataclass(frozen=True)
class CooBlock:
    rows: np.ndarray   # u32, global source states, ascending
    cols: np.ndarray   # u32, global successors, ascending within a row, SINK last
    vals: np.ndarray   # f64 probabilities count / N_rv
    nnz: int


@dataclass(frozen=True)
class SparseModel:
    """blocks[a][t]; rewards[a*N_g + s]; n_states = N_g + 1 (SINK)."""

    blocks: list
    rewards: np.ndarray
    n_states: int
    n_actions: int
    nt: int

    @property
    def n_nonsink_states(self) -> int:
        return self.n_states - 1

    def nnz_total(self) -> int:
        return sum(b.nnz for row in self.blocks for b in row)


def action_tables(actions) -> tuple:
    """(vectors [A,2], speeds [A]) with the reference's Python-float math."""
    if hasattr(actions, "vectors") and hasattr(actions, "speeds"):
        return np.asarray(actions.vectors(), dtype=np.float64), np.asarray(actions.speeds(), dtype=np.float64)
    return ActionSpace(actions.n_headings, actions.n_speeds, actions.f_max).vectors(), \
        ActionSpace(actions.n_headings, actions.n_speeds, actions.f_max).speeds()


class StepContext:
    """Everything one kinematic step needs (model_builder.py:185-259).

    The reference precomputes per-time obstacle gates on the host; here the
    gate is a summed-area-table box query evaluated inside the build kernel,
    with the same radius (see builder.gate_radius)."""

    def __init__(self, env, actions, rcfg, target):
        grid = env.grid
        ti, tj = int(target[0]), int(target[1])
        _require(0 <= ti < grid.nx and 0 <= tj < grid.ny, f"target cell {target} outside grid")
        self.env = env
        self.grid = grid
        self.actions = actions
        self.rcfg = rcfg
        self.target = (ti, tj)
        self.target_cell = tj * grid.nx + ti
        self.act_vecs, self.act_speeds = action_tables(actions)
        self._device_env = None   # lazily uploaded inputs (builder.DeviceEnv)

    def device_env(self, device=None):
        from .builder import DeviceEnv
        if self._device_env is None:
            self._device_env = DeviceEnv.from_host(self.env, device=device)
        return self._device_env


# ---------------------------------------------------------------------------
# solve
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SolverConfig:
    epsilon: float = 1e-8
    max_iterations: int | None = None

    def __post_init__(self):
        _require(self.epsilon > 0, "epsilon must be > 0")
        _require(self.max_iterations is None or self.max_iterations >= 1, "max_iterations must be >= 1")


@dataclass(frozen=True)
class PolicyValue:
    values: np.ndarray       # f64 [n_states], SINK last (0)
    actions: np.ndarray      # u16 [n_states - 1]
    iterations_run: int
    residual: float
    converged: bool
