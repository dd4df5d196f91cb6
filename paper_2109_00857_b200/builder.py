"""Model build on the B200: the drop-in for model_builder.compute_subgrid /
build_model (/root/reference/pkg/src/flowmdp/model_builder.py:376-580).

Host code here only marshals: it uploads the environment once
(``DeviceEnv``), derives the per-action constants with the reference's
Python-float arithmetic, allocates the device model and calls the C ABI.
All per-(state, action, realization) work runs in ``k_build``.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core_types import (
    OBJECTIVE_CODE,
    CooBlock,
    SparseModel,
    SubGridSpec,
    action_tables,
)
from .errors import ContractViolation


def _torch():
    import torch
    return torch


# ---------------------------------------------------------------------------
# device-resident inputs
# ---------------------------------------------------------------------------

@dataclass
class DeviceEnv:
    """Environment arrays resident in HBM (f64 / u8, reference layouts) plus
    the per-layer obstacle summed-area tables used for box queries."""

    grid: object
    mean: object
    modes: object
    coeffs: object
    g: object
    mask: object
    sat: object
    n_modes: int
    n_real: int
    _vbound: dict = field(default_factory=dict)
    _vmax: tuple | None = None
    _acts: dict = field(default_factory=dict)
    _scan: tuple | None = None   # (device maxima, j_range) of a scan done during upload
    _bounds_dev: tuple | None = None   # (device lo/hi bounds [4], j_range) of a bounds scan (upload)
    _vproof: tuple | None = None       # upper bounds of max|v_c| valid for the build's proofs
    envelope: object = None      # int32 [nt][N_c][4] per-cell velocity envelope (fm_velocity_scan)
    _env_rows: tuple | None = None   # rows [j0, j1) whose envelope is current (all layers)

    def _envelope_buf(self):
        if self.envelope is None:
            torch = _torch()
            g = self.grid
            self.envelope = torch.empty((g.nt, g.nx * g.ny, 4), dtype=torch.int32, device=self.mean.device)
        return self.envelope

    def envelope_for(self, j0: int, j1: int):
        """Device pointer of the envelope if it covers rows [j0, j1), else None."""
        if self._env_rows is not None and self._env_rows[0] <= j0 and j1 <= self._env_rows[1]:
            return self.envelope.data_ptr()
        return None

    def action_table(self, recs: np.ndarray):
        """Device copy of an action-record table (cached by content)."""
        key = recs.tobytes()
        if key not in self._acts:
            torch = _torch()
            self._acts[key] = torch.from_numpy(np.array(recs)).to(self.mean.device)
        return self._acts[key]

    @classmethod
    def from_host(cls, env, device=None, non_blocking: bool = False):
        """Upload an Environment (reference or mirror types).  numpy arrays,
        or (pinned) CPU torch tensors for non_blocking H2D."""
        torch = _torch()
        _lib.load()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

        def up(a, dtype):
            t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
            return t.to(device=dev, dtype=dtype, non_blocking=non_blocking).contiguous()

        grid, fld = env.grid, env.field
        mask_src = env.obstacles.mask
        if isinstance(mask_src, np.ndarray):
            mask_src = mask_src.view(np.uint8) if mask_src.dtype == np.bool_ else mask_src.astype(np.uint8)
        de = cls(
            grid=grid,
            mean=up(fld.mean, torch.float64),
            modes=up(fld.modes, torch.float64),
            coeffs=up(fld.coeffs, torch.float64),
            g=up(env.scalar.g_mean, torch.float64),
            mask=up(mask_src, torch.uint8),
            sat=None,
            n_modes=int(fld.modes.shape[0]),
            n_real=int(fld.coeffs.shape[1]),
        )
        de._make_sat()
        return de

    @classmethod
    def from_host_scanned(cls, env, slabs: int = 8, j_range: tuple | None = None, device=None):
        """Upload in time slabs on a copy stream and run compute_subgrid's
        exact scan (fm_velocity_max_slab) on each slab as soon as it lands,
        so the scan overlaps the rest of the host->device transfer.  The
        maxima stay on the device until ``velocity_max`` reads them (with
        ``j_range``: this rank's strip only, combined there by all-reduce).
        Inputs: numpy arrays or CPU torch tensors (pinned for a real overlap)."""
        torch = _torch()
        _lib.load()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        grid, fld = env.grid, env.field

        def host(a):
            return a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))

        mask_src = env.obstacles.mask
        if isinstance(mask_src, np.ndarray):
            mask_src = mask_src.view(np.uint8) if mask_src.dtype == np.bool_ else mask_src.astype(np.uint8)
        src = {"mean": host(fld.mean), "modes": host(fld.modes), "coeffs": host(fld.coeffs),
               "g": host(env.scalar.g_mean), "mask": host(mask_src)}
        dt = {"mean": torch.float64, "modes": torch.float64, "coeffs": torch.float64, "g": torch.float64,
              "mask": torch.uint8}
        for k, v in src.items():
            if v.dtype != dt[k] or not v.is_contiguous():
                src[k] = v.to(dt[k]).contiguous()
        dst = {k: torch.empty(v.shape, dtype=dt[k], device=dev) for k, v in src.items()}
        de = cls(grid=grid, mean=dst["mean"], modes=dst["modes"], coeffs=dst["coeffs"], g=dst["g"],
                 mask=dst["mask"], sat=None, n_modes=int(src["modes"].shape[0]), n_real=int(src["coeffs"].shape[1]))
        out = torch.zeros(4, dtype=torch.float64, device=dev)   # fm_velocity_bounds: lo/hi per component
        j0, j1 = j_range if j_range is not None else (0, grid.ny)
        main = torch.cuda.current_stream(dev)
        copy = torch.cuda.Stream(dev)
        copy.wait_stream(main)                       # the destination allocations
        nt = grid.nt
        bounds = [nt * i // max(1, min(slabs, nt)) for i in range(max(1, min(slabs, nt)) + 1)]
        lib = _lib.load()
        env_ptr = de._envelope_buf().data_ptr()
        for t0, t1 in zip(bounds[:-1], bounds[1:]):
            with torch.cuda.stream(copy):
                dst["mean"][t0:t1].copy_(src["mean"][t0:t1], non_blocking=True)
                for m in range(de.n_modes):          # [m][t] slabs: one contiguous run per mode
                    dst["modes"][m, t0:t1].copy_(src["modes"][m, t0:t1], non_blocking=True)
                dst["coeffs"][t0:t1].copy_(src["coeffs"][t0:t1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
            main.wait_event(ev)
            _lib.check(lib.fm_velocity_bounds(de.fm_grid(), de.fm_env(), int(t0), int(t1), int(j0), int(j1),
                                              out.data_ptr(), env_ptr, _lib.stream_ptr(main)), "fm_velocity_bounds")
        with torch.cuda.stream(copy):
            dst["g"].copy_(src["g"], non_blocking=True)
            dst["mask"].copy_(src["mask"], non_blocking=True)
        main.wait_stream(copy)
        for v in dst.values():                       # written on the copy stream, used on main
            v.record_stream(copy)
        de._make_sat()
        de._bounds_dev = (out, tuple(j_range) if j_range is not None else None)
        de._env_rows = (int(j0), int(j1))
        return de

    def _make_sat(self):
        torch = _torch()
        g = self.grid
        self.sat = torch.empty((g.nt, g.ny + 1, g.nx + 1), dtype=torch.int32, device=self.mean.device)
        _lib.check(_lib.load().fm_mask_sat(self.mask.data_ptr(), g.nt, g.ny, g.nx, self.sat.data_ptr(),
                                           _lib.stream_ptr()), "fm_mask_sat")

    # -- C structs ---------------------------------------------------------
    def fm_grid(self) -> _lib.FmGrid:
        g = self.grid
        return _lib.FmGrid(g.nx, g.ny, g.nt, float(g.dx), float(g.dt), float(g.origin[0]), float(g.origin[1]))

    def fm_env(self) -> _lib.FmEnv:
        return _lib.FmEnv(self.mean.data_ptr(), self.modes.data_ptr(), self.coeffs.data_ptr(),
                          self.g.data_ptr(), self.mask.data_ptr(), self.n_modes, self.n_real)

    # -- velocity statistics ------------------------------------------------
    def reset_derived(self):
        """Forget cached sub-grid / gate statistics (they are recomputed)."""
        self._vmax = None
        self._vbound = {}
        self._scan = None
        self._bounds_dev = None
        self._vproof = None
        self._env_rows = None

    def velocity_max(self, j_range: tuple | None = None, group=None) -> tuple:
        """Exact max |v_x|, |v_y| over (t, r, cell) -- compute_subgrid's scan.

        With ``j_range`` (this rank's row strip) and a process ``group``
        each rank scans its strip and the maxima are combined with one
        all-reduce (MAX) -- the same value as the full scan."""
        if self._vmax is None and self._scan is not None and self._scan[1] == (
                tuple(j_range) if j_range is not None else None):
            out, scanned_rows = self._scan   # scanned slab by slab during the upload
            self._scan = None
            if scanned_rows is not None and (group is not None or _dist_world() > 1):
                from .sharding import all_reduce_max
                all_reduce_max(out, group)
            h = out.cpu().numpy()
            if scanned_rows is not None and not (group is not None or _dist_world() > 1):
                return (float(h[0]), float(h[1]))   # a strip's maximum alone: never cached
            self._vmax = (float(h[0]), float(h[1]))
        if self._vmax is None:
            torch = _torch()
            out = torch.zeros(2, dtype=torch.float64, device=self.mean.device)
            # the scan also writes the per-cell envelope the build bins against
            r0, r1 = (0, self.grid.ny) if j_range is None else (int(j_range[0]), int(j_range[1]))
            _lib.check(_lib.load().fm_velocity_scan(self.fm_grid(), self.fm_env(), 0, self.grid.nt, r0, r1,
                                                    out.data_ptr(), self._envelope_buf().data_ptr(),
                                                    _lib.stream_ptr()), "fm_velocity_scan")
            self._env_rows = (r0, r1)
            if j_range is not None:
                if group is not None or _dist_world() > 1:
                    from .sharding import all_reduce_max
                    all_reduce_max(out, group)   # non-negative: max of maxima
                else:
                    # a strip's maximum alone is not the field's: never cached
                    # (the build's proofs rely on the cached value being global)
                    h = out.cpu().numpy()
                    return (float(h[0]), float(h[1]))
            h = out.cpu().numpy()
            self._vmax = (float(h[0]), float(h[1]))
        return self._vmax

    def subgrid(self, f_max: float, buffer: int = 1, j_range: tuple | None = None, group=None) -> SubGridSpec:
        """compute_subgrid's half widths (model_builder.py:376-399) from the
        envelope scan's bounds lo <= max|v_c| <= hi (fm_velocity_bounds; the
        per-cell envelope the build bins against is written on the way):
        ceil((v + f_max) dt / dx) is monotone in v, so when lo and hi give
        the same half width it is the exact one, and hi serves the build's
        proofs (an upper bound suffices there).  Otherwise -- or with a
        non-finite input -- the exact scan (velocity_max) decides.  With
        ``j_range`` / ``group``: this rank's strip, combined by all-reduce."""
        if buffer < 1:
            raise ContractViolation("buffer must be >= 1")
        if self._vmax is not None:
            return subgrid_from_vmax(self._vmax, f_max, self.grid, buffer)
        torch = _torch()
        key = tuple(j_range) if j_range is not None else None
        if self._bounds_dev is not None and self._bounds_dev[1] == key:
            out = self._bounds_dev[0]
        else:
            out = torch.zeros(4, dtype=torch.float64, device=self.mean.device)
            r0, r1 = (0, self.grid.ny) if j_range is None else (int(j_range[0]), int(j_range[1]))
            _lib.check(_lib.load().fm_velocity_bounds(self.fm_grid(), self.fm_env(), 0, self.grid.nt, r0, r1,
                                                      out.data_ptr(), self._envelope_buf().data_ptr(),
                                                      _lib.stream_ptr()), "fm_velocity_bounds")
            self._env_rows = (r0, r1)
        self._bounds_dev = None
        multi = group is not None or _dist_world() > 1
        if j_range is not None and multi:
            from .sharding import all_reduce_max
            all_reduce_max(out, group)   # non-negative: max of maxima (+inf stays)
        lox, hix, loy, hiy = (float(x) for x in out.cpu().numpy())
        if all(math.isfinite(v) for v in (hix, hiy)):
            lo = subgrid_from_vmax((lox, loy), f_max, self.grid, buffer)
            hi = subgrid_from_vmax((hix, hiy), f_max, self.grid, buffer)
            if lo == hi:
                if j_range is None or multi:   # a strip's bounds alone are not the field's
                    self._vproof = (hix, hiy)
                return hi
        return subgrid_from_vmax(self.velocity_max(j_range=j_range, group=group), f_max, self.grid, buffer)

    def proof_vmax(self) -> tuple:
        """Upper bounds of max|v_x|, max|v_y| for fm_build's proofs: the exact
        maxima when known, else the bounds of the last subgrid() call."""
        if self._vmax is not None:
            return self._vmax
        if self._vproof is not None:
            return self._vproof
        return self.velocity_max()

    def _maxima(self):
        """Device max-abs reductions behind velocity_bound (environment.py:404-419):
        max|mean| [nt][2], max|coeff| [nt][n_modes], max|mode| [n_modes][nt][2]."""
        if "mx" not in self._vbound:
            torch = _torch()
            g, nm, nr = self.grid, self.n_modes, self.n_real
            nc = g.nx * g.ny
            L = _lib.load()
            s = _lib.stream_ptr()
            dev = self.mean.device
            mean_mx = torch.empty(g.nt * 2, dtype=torch.float64, device=dev)
            _lib.check(L.fm_maxabs_segments(self.mean.data_ptr(), g.nt * 2, nc, 2, 2, nc * 2, 1,
                                            mean_mx.data_ptr(), s), "maxabs mean")
            coef_mx = torch.zeros(max(g.nt * nm, 1), dtype=torch.float64, device=dev)
            mode_mx = torch.zeros(max(nm * g.nt * 2, 1), dtype=torch.float64, device=dev)
            if nm:
                _lib.check(L.fm_maxabs_segments(self.coeffs.data_ptr(), g.nt * nm, nr, nm, nm, nr * nm, 1,
                                                coef_mx.data_ptr(), s), "maxabs coeffs")
                _lib.check(L.fm_maxabs_segments(self.modes.data_ptr(), nm * g.nt * 2, nc, 2, 2, nc * 2, 1,
                                                mode_mx.data_ptr(), s), "maxabs modes")
            self._vbound["mx"] = (mean_mx, coef_mx, mode_mx)
        return self._vbound["mx"]

    def gate_radius_device(self, f_max: float):
        """(rx, ry) of the obstacle gate as a device int32[2], no host round trip."""
        key = ("gate", float(f_max))
        if key not in self._vbound:
            torch = _torch()
            mean_mx, coef_mx, mode_mx = self._maxima()
            out = torch.empty(2, dtype=torch.int32, device=self.mean.device)
            _lib.check(_lib.load().fm_gate_radius(self.fm_grid(), mean_mx.data_ptr(), coef_mx.data_ptr(),
                                                  mode_mx.data_ptr(), self.n_modes, float(f_max), out.data_ptr(),
                                                  None, _lib.stream_ptr()), "fm_gate_radius")
            self._vbound[key] = out
        return self._vbound[key]

    def velocity_bound(self) -> tuple:
        """Triangle bound of environment.py:404-419: device max-abs
        reductions, then the reference's per-t combination on the host."""
        if "b" not in self._vbound:
            g, nm = self.grid, self.n_modes
            mean_mx, coef_mx, mode_mx = self._maxima()
            mean_mx = mean_mx.cpu().numpy().reshape(g.nt, 2)
            coef_mx = coef_mx.cpu().numpy()[: g.nt * nm].reshape(g.nt, nm)
            mode_mx = mode_mx.cpu().numpy()[: nm * g.nt * 2].reshape(nm, g.nt, 2)
            bounds = []
            for c in (0, 1):
                per_t = mean_mx[:, c].copy()
                for m in range(nm):
                    per_t = per_t + coef_mx[:, m] * mode_mx[m, :, c]
                bounds.append(float(per_t.max()))
            self._vbound["b"] = (bounds[0], bounds[1])
        return self._vbound["b"]


def _dist_world() -> int:
    try:
        import torch.distributed as dist
        return dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    except Exception:
        return 1


def gate_radius(denv: DeviceEnv, f_max: float) -> tuple:
    """Obstacle-gate dilation radius in cells (model_builder.py:218-223)."""
    bx, by = denv.velocity_bound()
    g = denv.grid
    rx = int(math.ceil((bx + f_max) * g.dt / g.dx)) + 1
    ry = int(math.ceil((by + f_max) * g.dt / g.dx)) + 1
    return rx, ry


def subgrid_from_vmax(vmax: tuple, f_max: float, grid, buffer: int = 1) -> SubGridSpec:
    """half_width = ceil((max|v_c| + f_max) * dt / dx) + buffer (model_builder.py:397-399)."""
    if buffer < 1:
        raise ContractViolation("buffer must be >= 1")
    hx = int(math.ceil((vmax[0] + f_max) * grid.dt / grid.dx)) + buffer
    hy = int(math.ceil((vmax[1] + f_max) * grid.dt / grid.dx)) + buffer
    return SubGridSpec(half_width_x=hx, half_width_y=hy)


def compute_subgrid(field, actions, grid, buffer: int = 1, device_env: DeviceEnv | None = None) -> SubGridSpec:
    """Drop-in for model_builder.compute_subgrid (model_builder.py:376-399).

    The max over every (t, realization, cell) runs in ``k_vmax``: the f32
    envelope's bounds decide the half widths when unambiguous, else the
    exact f64 scan (DeviceEnv.subgrid)."""
    if buffer < 1:
        raise ContractViolation("buffer must be >= 1")
    denv = device_env
    if denv is None:
        env = _FieldOnly(grid, field)
        denv = DeviceEnv.from_host(env)
    return denv.subgrid(actions.f_max, buffer)


class _FieldOnly:
    """Environment stand-in for compute_subgrid(field, ...) calls."""

    def __init__(self, grid, field):
        nt, ny, nx = field.mean.shape[:3]
        self.grid = grid
        self.field = field
        self.scalar = type("S", (), {"g_mean": np.zeros((nt, ny, nx))})()
        self.obstacles = type("O", (), {"mask": np.zeros((nt, ny, nx), dtype=bool)})()


# ---------------------------------------------------------------------------
# device model
# ---------------------------------------------------------------------------

def action_records(actions, rcfg, grid) -> np.ndarray:
    """Per-action constants with the reference's rounding (model_builder.py:350-358)."""
    vec, spd = action_tables(actions)
    recs = np.zeros((vec.shape[0], 6), dtype=np.float64)
    dt = float(grid.dt)
    for a in range(vec.shape[0]):
        f = float(spd[a])
        neg_cff = -(rcfg.c_f * f * f)
        if rcfg.objective == "time":
            base = -dt
        else:
            base = -(rcfg.c_f * f * f) * dt
        recs[a] = (vec[a, 0], vec[a, 1], base, base + rcfg.r_term, neg_cff, 0.0)
    return recs


@dataclass
class DeviceModel:
    """Compact model in HBM (see fm_model in include/flowmdp_b200.h)."""

    grid: object
    n_actions: int
    n_real: int
    subgrid: SubGridSpec
    row_ptr: object      # int64  [n_rows]
    row_nnz: object      # int16  [n_rows] (u16 bits)
    reward: object       # f64    [n_rows]
    entries: object      # int32  [capacity] (u32 bits)
    d_nnz: object        # int64  [1]
    nnz: int
    t_range: tuple
    j_range: tuple

    @property
    def cell0(self) -> int:
        """First cell whose rows the model holds (row strip j_range)."""
        return self.j_range[0] * self.grid.nx

    @property
    def ncell(self) -> int:
        return (self.j_range[1] - self.j_range[0]) * self.grid.nx

    @property
    def n_rows(self) -> int:
        """Rows (t, c, a) of every layer for the strip's cells only:
        row id = (t * ncell + c - cell0) * n_actions + a."""
        return self.grid.nt * self.ncell * self.n_actions

    def row_ids(self, t: int, a: int, j0: int, j1: int):
        """Device row ids of action a, layer t, source rows j in [j0, j1)."""
        torch = _torch()
        g = self.grid
        if not (self.j_range[0] <= j0 and j1 <= self.j_range[1]):
            raise ContractViolation(f"rows [{j0}, {j1}) are not in this model (rows {self.j_range})")
        cells = torch.arange(j0 * g.nx, j1 * g.nx, device=self.row_ptr.device, dtype=torch.int64)
        return cells, (t * self.ncell + cells - self.cell0) * self.n_actions + a

    @property
    def nt(self) -> int:
        return self.grid.nt

    @property
    def n_states(self) -> int:
        return self.grid.nt * self.grid.nx * self.grid.ny + 1

    _pending: tuple | None = None
    _scratch: tuple | None = None
    group_events: list = field(default_factory=list)   # ((t0, t1), cuda event) per launch group
    group_nnz: object = None   # pinned int64 [groups]: the entry counter after each group

    def host_buffers(self) -> dict:
        """Pinned host buffers for stream_to_host / copy_to_host."""
        torch = _torch()
        return {"row_ptr": torch.empty(self.row_ptr.numel(), dtype=torch.int64).pin_memory(),
                "row_nnz": torch.empty(self.row_nnz.numel(), dtype=torch.int16).pin_memory(),
                "reward": torch.empty(self.reward.numel(), dtype=torch.float64).pin_memory(),
                "entries": torch.empty(int(self.entries.numel()), dtype=torch.int32).pin_memory()}

    def stream_to_host(self, host: dict, stream) -> int:
        """Copy the compact model to pinned host buffers while the build is
        still running: for each slab group (launch order), wait for its
        build on the host, then queue the D2H of its rows (row pointers,
        entry counts, rewards: one contiguous range per group) and of the
        entries it appended (bump-allocated: [counter before, counter
        after)) on ``stream``.  Without groups: one copy after the build.
        Returns the bytes copied.  If check() later reports a rebuild
        (capacity), the caller must copy again (copy_to_host)."""
        torch = _torch()
        if not self.group_events or self.group_nnz is None:
            stream.wait_stream(torch.cuda.current_stream())
            return self.copy_to_host(host, stream)
        g, na = self.grid, self.n_actions
        cap = int(self.entries.numel())
        prev, nbytes = 0, 0
        for k, ((g0, g1), ev) in enumerate(self.group_events):
            ev.synchronize()
            end = min(int(self.group_nnz[k]), cap)
            r0, r1 = g0 * self.ncell * na, g1 * self.ncell * na
            stream.wait_event(ev)
            with torch.cuda.stream(stream):
                for key in ("row_ptr", "row_nnz", "reward"):
                    src = getattr(self, key)[r0:r1]
                    host[key][r0:r1].copy_(src, non_blocking=True)
                    nbytes += src.numel() * src.element_size()
                if end > prev:
                    host["entries"][prev:end].copy_(self.entries[prev:end], non_blocking=True)
                    nbytes += (end - prev) * 4
            prev = max(prev, end)
        return nbytes

    def copy_to_host(self, host: dict, stream) -> int:
        """The whole compact model to pinned host buffers on ``stream``
        (after check()); returns the bytes copied."""
        torch = _torch()
        self.check()
        nbytes = 0
        with torch.cuda.stream(stream):
            for key in ("row_ptr", "row_nnz", "reward"):
                src = getattr(self, key)
                host[key].copy_(src, non_blocking=True)
                nbytes += src.numel() * src.element_size()
            if host["entries"].numel() < self.nnz:
                host["entries"] = torch.empty(int(self.entries.numel()), dtype=torch.int32).pin_memory()
            host["entries"][: self.nnz].copy_(self.entries[: self.nnz], non_blocking=True)
            nbytes += self.nnz * 4
        return nbytes

    def check(self) -> bool:
        """Finish a (deferred) build: census, sub-grid overflow (raises the
        reference's ContractViolation), capacity.  Returns True if the model
        had to be rebuilt with a larger entry buffer (consumers queued after
        the launch must then be re-run)."""
        if self._pending is None:
            return False
        args, keep = self._pending
        L = _lib.load()
        rebuilt = False
        for _attempt in range(2):
            m = self.fm_model()
            needed = C.c_uint64(0)
            vio = _lib.FmViolation()
            st = L.fm_build_check(C.byref(args), C.byref(m), C.byref(needed), C.byref(vio), _lib.stream_ptr())
            if st == _lib.FM_CAPACITY:
                torch = _torch()
                self.entries = torch.empty(int(needed.value) + 1024, dtype=torch.int32, device=self.entries.device)
                self.d_nnz.zero_()
                keep[2].zero_()
                m = self.fm_model()
                _lib.check(L.fm_build_launch(C.byref(args), C.byref(m), _lib.stream_ptr()), "fm_build_launch")
                rebuilt = True
                continue
            _lib.check(st, "fm_build")
            self.nnz = int(needed.value)
            self._pending = None
            return rebuilt
        raise RuntimeError("fm_build: capacity retry failed")

    def fm_model(self) -> _lib.FmModel:
        g = self.grid
        return _lib.FmModel(g.nx, g.ny, g.nt, self.n_actions, self.n_real,
                            self.subgrid.half_width_x, self.subgrid.half_width_y,
                            self.cell0, self.ncell, self.n_rows, self.row_ptr.data_ptr(), self.row_nnz.data_ptr(),
                            self.reward.data_ptr(), self.entries.data_ptr(),
                            int(self.entries.numel()), self.d_nnz.data_ptr())

    def rows_coo(self, t: int, a: int, j0: int, j1: int):
        """Canonical COO of action a, layer t, source rows j in [j0, j1) (host
        arrays rows u32, cols u32, vals f64, rewards f64 per cell) gathered
        from the compact model -- for spot checks of models too large to
        export whole."""
        torch = _torch()
        self.check()
        g, na = self.grid, self.n_actions
        nc = g.nx * g.ny
        cells, rid = self.row_ids(t, a, j0, j1)
        ptr = self.row_ptr[rid]
        cnt = self.row_nnz[rid].to(torch.int64) & 0xFFFF
        idx = torch.repeat_interleave(ptr, cnt) + (torch.arange(int(cnt.sum()), device=ptr.device)
                                                   - torch.repeat_interleave(torch.cumsum(cnt, 0) - cnt, cnt))
        ent = self.entries[idx].to(torch.int64) & 0xFFFFFFFF
        src = torch.repeat_interleave(cells, cnt)
        slot, count = ent >> 16, ent & 0xFFFF
        hx, hy = self.subgrid.half_width_x, self.subgrid.half_width_y
        W = 2 * hx + 1
        nslot = W * (2 * hy + 1)
        di, dj = slot % W - hx, slot // W - hy
        col = (t + 1) * nc + (src // g.nx + dj) * g.nx + (src % g.nx + di)
        col = torch.where(slot == nslot, torch.full_like(col, g.nt * nc), col)
        rows = (t * nc + src).cpu().numpy().astype(np.uint32)
        # true division on the host (a device tensor / scalar may multiply by the reciprocal)
        vals = count.cpu().numpy().astype(np.float64) / float(self.n_real)
        return rows, col.cpu().numpy().astype(np.uint32), vals, self.reward[rid].cpu().numpy()

    def export_device(self):
        """Canonical COO on the device: (block_off, rows, cols, vals, rewards)."""
        torch = _torch()
        self.check()   # a deferred build: census (nnz sizes the outputs), overflow, capacity
        dev = self.reward.device
        nb = self.n_actions * self.grid.nt
        scratch = torch.empty(self.n_rows + 1, dtype=torch.int64, device=dev)
        block_off = torch.zeros(nb + 1, dtype=torch.int64, device=dev)
        rows = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev)
        cols = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev)
        vals = torch.empty(max(self.nnz, 1), dtype=torch.float64, device=dev)
        rewards = torch.empty(self.n_rows, dtype=torch.float64, device=dev)
        m = self.fm_model()
        _lib.check(_lib.load().fm_export_coo(C.byref(m), scratch.data_ptr(), block_off.data_ptr(),
                                             rows.data_ptr(), cols.data_ptr(), vals.data_ptr(),
                                             rewards.data_ptr(), _lib.stream_ptr()), "fm_export_coo")
        return block_off, rows[: self.nnz], cols[: self.nnz], vals[: self.nnz], rewards

    def to_sparse_model(self) -> SparseModel:
        """D2H into the reference's SparseModel (blocks[a][t] CooBlocks)."""
        if self.t_range != (0, self.grid.nt) or self.j_range != (0, self.grid.ny):
            raise ContractViolation("to_sparse_model needs a full (unsharded) model")
        block_off, rows, cols, vals, rewards = self.export_device()
        off = block_off.cpu().numpy()
        rows_h = rows.cpu().numpy().view(np.uint32)
        cols_h = cols.cpu().numpy().view(np.uint32)
        vals_h = vals.cpu().numpy()
        rew_h = rewards.cpu().numpy()
        nt, na = self.grid.nt, self.n_actions
        blocks = []
        for a in range(na):
            row = []
            for t in range(nt):
                lo, hi = int(off[a * nt + t]), int(off[a * nt + t + 1])
                row.append(CooBlock(rows=rows_h[lo:hi], cols=cols_h[lo:hi], vals=vals_h[lo:hi], nnz=hi - lo))
            blocks.append(row)
        return SparseModel(blocks=blocks, rewards=rew_h, n_states=self.n_states, n_actions=na, nt=nt)


def build_device_model(denv: DeviceEnv, actions, rcfg, target, subgrid: SubGridSpec,
                       t_range: tuple | None = None, j_range: tuple | None = None,
                       capacity_hint: int | None = None, defer_check: bool = False,
                       lean: bool = True, reuse: DeviceModel | None = None,
                       t_groups: list | None = None, reserve_sms: int = 0,
                       reward_sum: str = "sequential") -> DeviceModel:
    """Run K_build over slabs t_range x row strip j_range; the model stays in HBM.

    ``reward_sum``: "sequential" (default) -- row rewards are the
    reference's ascending-realization f64 sum (model_builder.py:457-458),
    bit-exact; "counts" -- formed from the per-slot counts whenever the fast
    path is proven (fm_build_args.reward_mode 1): counts, columns and
    probabilities stay bit-exact, rewards agree to rounding (~1e-13
    relative; north_star's tolerance is 1e-5) and net-energy rows take the
    binned build.

    With defer_check the kernel is only enqueued: consumers (the backward
    solve) can be queued behind it and ``DeviceModel.check()`` performs the
    census / overflow / capacity check later (it rebuilds on a capacity
    miss and returns True when it did).

    ``lean=False`` withholds the exact velocity maxima and the host action
    table, so every transition takes the fully checked path (same output;
    the parity tests use it to cover both paths).

    ``reuse`` hands over the buffers of a previous model of the same problem
    shape (that model must not be used afterwards): repeated planner steps
    then allocate nothing.

    ``t_groups`` (slab ranges covering t_range, in launch order -- for the
    pipelined solve, descending): one launch per group on the current
    stream, an event recorded after each (``DeviceModel.group_events``), so
    a solve stream can start on a group's layers while later groups build;
    ``reserve_sms`` leaves that many SMs' worth of blocks free for it."""
    torch = _torch()
    L = _lib.load()
    grid = denv.grid
    ti, tj = int(target[0]), int(target[1])
    if not (0 <= ti < grid.nx and 0 <= tj < grid.ny):
        raise ContractViolation(f"target cell {tuple(target)} outside grid")
    t0, t1 = t_range if t_range is not None else (0, grid.nt)
    j0, j1 = j_range if j_range is not None else (0, grid.ny)
    full = (t0, t1) == (0, grid.nt)   # every row of the strip is written
    dev = denv.mean.device
    recs = action_records(actions, rcfg, grid)
    na = recs.shape[0]
    d_act = denv.action_table(recs)
    d_gate = denv.gate_radius_device(float(actions.f_max))
    hx, hy = subgrid.half_width_x, subgrid.half_width_y
    nc = grid.nx * grid.ny
    n_rows = grid.nt * (j1 - j0) * grid.nx * na   # the strip's rows only (all layers)
    active_rows = (t1 - t0) * (j1 - j0) * grid.nx * na
    n_slot1 = (2 * hx + 1) * (2 * hy + 1) + 1
    cap = capacity_hint if capacity_hint else active_rows * min(n_slot1, denv.n_real, 6) + 1024
    if reuse is not None and reuse.row_ptr.numel() == n_rows and reuse.row_ptr.device == dev and \
            reuse.j_range == (j0, j1):
        row_ptr, row_nnz, reward, d_nnz = reuse.row_ptr, reuse.row_nnz, reuse.reward, reuse.d_nnz
        d_nnz.zero_()
        if not full:
            row_nnz.zero_()
            reward.zero_()
        entries = reuse.entries if reuse.entries.numel() >= cap else None
        viol, counter = reuse._scratch
        viol.zero_()
        reuse._pending = None
    else:
        alloc = torch.empty if full else torch.zeros
        row_ptr = torch.empty(n_rows, dtype=torch.int64, device=dev)
        row_nnz = alloc(n_rows, dtype=torch.int16, device=dev)
        reward = alloc(n_rows, dtype=torch.float64, device=dev)
        d_nnz = torch.zeros(1, dtype=torch.int64, device=dev)
        viol = torch.zeros(grid.nt * na, dtype=torch.int32, device=dev)
        counter = torch.zeros(1, dtype=torch.int32, device=dev)
        entries = None
    rw = _lib.FmReward(OBJECTIVE_CODE[rcfg.objective], float(rcfg.c_f), float(rcfg.c_r),
                       float(rcfg.r_term), float(rcfg.r_outbound), ti, tj)
    # the exact velocity maxima (when this env's sub-grid scan has run) let
    # the kernel prove the lean path's preconditions; they change no output
    vmx, vmy = denv.proof_vmax() if lean else (-1.0, -1.0)
    recs = np.ascontiguousarray(recs)
    args = _lib.FmBuildArgs(denv.fm_grid(), denv.fm_env(), rw, d_act.data_ptr(), na, hx, hy, 0, 0,
                            denv.sat.data_ptr(), t0, t1, j0, j1, viol.data_ptr(), counter.data_ptr(),
                            d_gate.data_ptr(), recs.ctypes.data if lean else None, vmx, vmy,
                            denv.envelope_for(j0, j1) if lean else None, int(reserve_sms))
    if reward_sum not in ("sequential", "counts"):
        raise ContractViolation(f"reward_sum must be 'sequential' or 'counts', not {reward_sum!r}")
    args.reward_mode = 1 if reward_sum == "counts" else 0
    if entries is None:
        entries = torch.empty(int(cap), dtype=torch.int32, device=dev)
    dm = DeviceModel(grid=grid, n_actions=na, n_real=denv.n_real, subgrid=subgrid,
                     row_ptr=row_ptr, row_nnz=row_nnz, reward=reward, entries=entries,
                     d_nnz=d_nnz, nnz=0, t_range=(t0, t1), j_range=(j0, j1))
    dm._pending = (args, (d_act, d_gate, viol, counter, denv, recs))
    dm._scratch = (viol, counter)
    m = dm.fm_model()
    dm.group_events = []
    if t_groups:
        if sorted(t for g in t_groups for t in range(*g)) != list(range(t0, t1)):
            raise ContractViolation("t_groups must partition the slab range")
        # the entry counter after each group, copied to pinned host memory
        # in stream order (stream_to_host reads it once the group's event fired)
        snap = getattr(reuse, "group_nnz", None) if reuse is not None else None
        if snap is None or snap.numel() < len(t_groups):
            snap = torch.zeros(len(t_groups), dtype=torch.int64).pin_memory()
        dm.group_nnz = snap
        # the obstacle tasks of the whole range first (the slow ones), then
        # the lean tasks group by group: each group completes with one short
        # launch (fm_build_args.phases); its entries follow the obstacle
        # launch's in the bump allocation
        oa = _lib.FmBuildArgs.from_buffer_copy(args)
        oa.phases = 2
        _lib.check(L.fm_build_launch(C.byref(oa), C.byref(m), _lib.stream_ptr()), "fm_build_launch")
        for k, (g0, g1) in enumerate(t_groups):
            ga = _lib.FmBuildArgs.from_buffer_copy(args)
            ga.t0, ga.t1 = int(g0), int(g1)
            ga.phases = 1
            _lib.check(L.fm_build_launch(C.byref(ga), C.byref(m), _lib.stream_ptr()), "fm_build_launch")
            snap[k:k + 1].copy_(d_nnz, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            dm.group_events.append(((int(g0), int(g1)), ev))
    else:
        _lib.check(L.fm_build_launch(C.byref(args), C.byref(m), _lib.stream_ptr()), "fm_build_launch")
    if not defer_check:
        dm.check()
    return dm


def build_model(ctx, subgrid: SubGridSpec, n_threads: int = 1) -> SparseModel:
    """Drop-in for model_builder.build_model (model_builder.py:532-580).

    ``n_threads`` is accepted for signature compatibility; the GPU build is
    deterministic and its output identical for any value."""
    del n_threads
    denv = ctx.device_env() if hasattr(ctx, "device_env") else DeviceEnv.from_host(ctx.env)
    dm = build_device_model(denv, ctx.actions, ctx.rcfg, ctx.target, subgrid)
    return dm.to_sparse_model()
