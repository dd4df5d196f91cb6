"""Synthetic inputs and named workloads for tests and the benchmark.

The reference generates its benchmark worlds with synthesis.py
(generate_double_gyre :163-215, generate_radiation :218-240,
generate_obstacles :243-264).  /root/reference is not present on the GPU
box, so this module re-derives the same fields from the same formulas and
the same numpy call sequence; on one machine the arrays are bit-identical
to the reference's (checked by tests/golden/make_golden.py, which records
input digests).  This is input generation, not part of the measured path.

Named workloads follow SURVEY.md section 8(d): smoke, desk (C1), C1-1k,
paper (C2), C3 (energy), C4 (net-energy, two obstacles), C5 (stress).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core_types import (
    ActionSpace,
    DOVelocityField,
    Environment,
    GridSpec,
    ObstacleMask,
    RewardConfig,
    ScalarMeanField,
)

TWO_PI = 2.0 * np.pi
# (p, q) streamfunction wavenumbers of the perturbation modes, in order
WAVENUMBERS = ((1, 1), (2, 1), (1, 2), (2, 2), (3, 1), (1, 3), (3, 2), (2, 3),
               (3, 3), (4, 1), (1, 4), (4, 2), (2, 4), (4, 3), (3, 4), (4, 4))


def _unit_centres(n: int) -> np.ndarray:
    return (np.arange(n, dtype=np.float64) + 0.5) / n


def double_gyre(grid: GridSpec, amplitude: float, eps: float, n_modes: int, n_realizations: int,
                seed: int) -> DOVelocityField:
    """Stochastic double gyre in DO form: modulated mean, Gram-Schmidt
    orthonormal perturbation modes, centred skewed-mixture coefficients."""
    assert 0 <= n_modes <= len(WAVENUMBERS)
    xh, yh = _unit_centres(grid.nx), _unit_centres(grid.ny)
    nt, ny, nx = grid.nt, grid.ny, grid.nx

    # mean: psi = sin(2 pi x) sin(pi y), strength modulated by 15% over the horizon
    gyre_u = np.sin(2.0 * np.pi * xh)[None, :] * np.cos(np.pi * yh)[:, None]
    gyre_v = -(2.0 * ny / nx) * np.cos(2.0 * np.pi * xh)[None, :] * np.sin(np.pi * yh)[:, None]
    mean = np.empty((nt, ny, nx, 2))
    for t in range(nt):
        strength = amplitude * (1.0 + 0.15 * np.sin(2.0 * np.pi * t / nt))
        mean[t, :, :, 0] = strength * gyre_u
        mean[t, :, :, 1] = strength * gyre_v

    modes = np.zeros((n_modes, nt, ny, nx, 2))
    for t in range(nt):
        raw = np.empty((n_modes, 2 * nx * ny))
        for m in range(n_modes):
            p, q = WAVENUMBERS[m]
            shift = 0.2 * np.sin(2.0 * np.pi * t / nt + 0.9 * m)
            arg_x = p * np.pi * xh + shift
            comp = np.empty((ny, nx, 2))
            comp[:, :, 0] = -q * np.sin(arg_x)[None, :] * np.cos(q * np.pi * yh)[:, None]
            comp[:, :, 1] = p * np.cos(arg_x)[None, :] * np.sin(q * np.pi * yh)[:, None]
            raw[m] = comp.reshape(-1)
        if n_modes:
            modes[:, t] = _gram_schmidt(raw).reshape(n_modes, ny, nx, 2)

    coeffs = np.zeros((nt, n_realizations, n_modes))
    if n_modes and eps > 0:
        rng = np.random.default_rng(seed)
        shape = (nt, n_realizations, n_modes)
        first = rng.random(shape) < 0.7
        lo = rng.normal(-0.5, 0.7, shape)
        hi = rng.normal(0.5 * 0.7 / 0.3, 1.3, shape)
        z = np.where(first, lo, hi)
        z -= z.mean(axis=1, keepdims=True)
        energy = np.sqrt(2.0 * nx * ny)
        for m in range(n_modes):
            decay = 0.65 ** m
            for t in range(nt):
                s = eps * energy * decay * (1.0 + 0.25 * np.sin(2.0 * np.pi * t / nt + 0.9 * m))
                coeffs[t, :, m] = s * z[t, :, m]
    return DOVelocityField(mean=mean, modes=modes, coeffs=coeffs)


def _gram_schmidt(rows: np.ndarray) -> np.ndarray:
    """Modified Gram-Schmidt with plain dot products, row by row."""
    out = rows.astype(np.float64).copy()
    for m in range(out.shape[0]):
        for k in range(m):
            out[m] -= (out[k] @ out[m]) * out[k]
        nrm = np.sqrt(out[m] @ out[m])
        if nrm < 1e-12:
            raise ValueError("degenerate perturbation mode")
        out[m] /= nrm
    return out


def radiation(grid: GridSpec, base_level: float, cloud_speed: float, cloud_width: float) -> ScalarMeanField:
    """Gaussian cloud dip entering at the east edge, drifting west."""
    w = cloud_width * grid.dx
    xc = grid.origin[0] + (np.arange(grid.nx, dtype=np.float64) + 0.5) * grid.dx
    east = grid.origin[0] + grid.nx * grid.dx
    g = np.empty((grid.nt, grid.ny, grid.nx))
    for t in range(grid.nt):
        centre = east - cloud_speed * grid.dx * t
        g[t] = (base_level * (1.0 - np.exp(-((xc - centre) ** 2) / (2.0 * w * w))))[None, :]
    return ScalarMeanField(g_mean=g)


def obstacles(grid: GridSpec, side: int, entry_time: float, speed: float, positions) -> ObstacleMask:
    """Squares moving east at `speed` cells/step, rasterised by rounding."""
    mask = np.zeros((grid.nt, grid.ny, grid.nx), dtype=bool)
    for t in range(grid.nt):
        if t < entry_time:
            continue
        for px, py in positions:
            i0 = int(np.rint(float(px) + speed * (t - entry_time)))
            j0 = int(np.rint(float(py)))
            ia, ib = max(i0, 0), min(i0 + side, grid.nx)
            ja, jb = max(j0, 0), min(j0 + side, grid.ny)
            if ia < ib and ja < jb:
                mask[t, ja:jb, ia:ib] = True
    return ObstacleMask(mask=mask)


# ---------------------------------------------------------------------------
# named workloads (pkg/configs/*.json)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Workload:
    name: str
    grid: GridSpec
    amplitude: float
    eps: float
    n_modes: int
    n_realizations: int
    seed: int
    radiation: tuple          # (base_level, cloud_speed, cloud_width)
    obstacles: tuple          # (side, entry_time, speed, positions)
    n_headings: int
    n_speeds: int
    f_max: float
    objective: str
    start: tuple
    target: tuple
    c_f: float = 1.0
    c_r: float = 0.5
    r_term: float = 100.0
    r_outbound: float = -300.0
    buffer: int = 1
    subgrid_hint: tuple | None = None   # exact (hx, hy), pinned by tests

    @property
    def n_actions(self) -> int:
        return self.n_headings * self.n_speeds

    @property
    def transitions(self) -> int:
        """U = N_c * nt * |A| * N_rv simulated one-step transitions."""
        g = self.grid
        return g.nx * g.ny * g.nt * self.n_actions * self.n_realizations

    def environment(self) -> Environment:
        g = self.grid
        return Environment(
            grid=g,
            field=double_gyre(g, self.amplitude, self.eps, self.n_modes, self.n_realizations, self.seed),
            scalar=radiation(g, *self.radiation),
            obstacles=obstacles(g, *self.obstacles),
        )

    def actions(self) -> ActionSpace:
        return ActionSpace(self.n_headings, self.n_speeds, self.f_max)

    def reward_config(self) -> RewardConfig:
        return RewardConfig(self.objective, c_f=self.c_f, c_r=self.c_r, r_term=self.r_term,
                            r_outbound=self.r_outbound)

    def with_(self, **kw) -> "Workload":
        d = dict(self.__dict__)
        d.update(kw)
        return Workload(**d)


def _wl(name, n, nt, n_rv, objective="time", heads=8, amp=0.4, side=6, pos=((22, 22),), width=6.0,
        start=None, target=None, dt=1.0, eps=0.12, n_modes=8, seed=42, **kw):
    g = GridSpec(nx=n, ny=n, nt=nt, dx=1.0, dt=dt)
    return Workload(name=name, grid=g, amplitude=amp, eps=eps, n_modes=n_modes, n_realizations=n_rv,
                    seed=seed, radiation=(1.5, 0.5, width), obstacles=(side, 0, 0.5, pos),
                    n_headings=heads, n_speeds=2, f_max=1.0, objective=objective,
                    start=start, target=target, **kw)


WORKLOADS = {
    # pkg/configs/smoke_env.json + smoke_run.json
    "smoke": Workload(name="smoke", grid=GridSpec(nx=9, ny=9, nt=10, dx=1.0, dt=0.8), amplitude=0.3,
                      eps=0.15, n_modes=4, n_realizations=32, seed=5, radiation=(1.0, 0.5, 3.0),
                      obstacles=(2, 0, 0.0, ((4, 4),)), n_headings=8, n_speeds=2, f_max=1.0,
                      objective="time", start=(2, 2), target=(6, 6)),
    # C1 desk: pkg/configs/desk_env.json + desk_run_*.json
    "desk": _wl("desk", 50, 60, 500, start=(25, 12), target=(25, 38), subgrid_hint=(4, 6)),
    "desk_energy": _wl("desk_energy", 50, 60, 500, "energy", start=(25, 12), target=(25, 38)),
    "desk_net_energy": _wl("desk_net_energy", 50, 60, 500, "net_energy", start=(25, 12), target=(25, 38)),
    "desk_1k": _wl("desk_1k", 50, 60, 1000, start=(25, 12), target=(25, 38)),
    # C2 paper-scale, time objective (BASELINE.json configs[1])
    "paper": _wl("paper", 100, 100, 5000, side=12, pos=((44, 44),), width=12.0, start=(50, 24), target=(50, 76),
                 subgrid_hint=(5, 5)),
    "paper_wide": _wl("paper_wide", 100, 100, 5000, amp=3.0, side=12, pos=((44, 44),), width=12.0,
                      start=(50, 24), target=(50, 76)),
    # C3 energy, C4 net-energy + two moving obstacles
    "paper_energy": _wl("paper_energy", 100, 100, 5000, "energy", side=12, pos=((44, 44),), width=12.0,
                        start=(50, 24), target=(50, 76)),
    "paper_net_energy": _wl("paper_net_energy", 100, 100, 5000, "net_energy", side=12,
                            pos=((44, 44), (10, 70)), width=12.0, start=(50, 24), target=(50, 76)),
    # C5 stress
    "stress": _wl("stress", 400, 200, 10000, heads=16, side=48, pos=((176, 176),), width=48.0,
                  start=(200, 96), target=(200, 304)),
}


def get(name: str) -> Workload:
    return WORKLOADS[name]
