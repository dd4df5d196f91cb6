"""Shared fixtures.  The world factories re-derive the reference test
fixtures (pkg/tests/conftest.py:26-128) with the same numpy call sequence,
so make_random_env(seed) here produces the same arrays as the reference's
(tests/test_oracle_golden.py checks the input digests)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.dirname(os.path.abspath(__file__))):
    if p not in sys.path:
        sys.path.insert(0, p)

from paper_2109_00857_b200.core_types import (  # noqa: E402
    OBJECTIVES,
    ActionSpace,
    DOVelocityField,
    Environment,
    GridSpec,
    ObstacleMask,
    RewardConfig,
    ScalarMeanField,
)
from paper_2109_00857_b200 import workloads  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the sm_100a extension")
    config.addinivalue_line("markers", "slow: minutes-scale case")


def make_tiny_env() -> Environment:
    """6x6x6 generated world, one static obstacle cell at (3, 3)."""
    g = GridSpec(nx=6, ny=6, nt=6, dx=1.0, dt=0.7)
    return Environment(
        grid=g,
        field=workloads.double_gyre(g, 0.3, 0.15, 3, 16, 7),
        scalar=workloads.radiation(g, 1.0, 0.5, 2.0),
        obstacles=workloads.obstacles(g, 1, 0, 0.0, ((3, 3),)),
    )


def make_zero_flow_env(nx=5, ny=5, nt=6, dx=1.0, dt=1.0, n_realizations=4, mask_cells=(), g_level=1.0):
    """Still water: successors are a pure function of the action."""
    g = GridSpec(nx=nx, ny=ny, nt=nt, dx=dx, dt=dt)
    mask = np.zeros((nt, ny, nx), dtype=bool)
    for ci, cj in mask_cells:
        mask[:, cj, ci] = True
    return Environment(
        grid=g,
        field=DOVelocityField(mean=np.zeros((nt, ny, nx, 2)), modes=np.zeros((0, nt, ny, nx, 2)),
                              coeffs=np.zeros((nt, n_realizations, 0))),
        scalar=ScalarMeanField(g_mean=np.full((nt, ny, nx), g_level)),
        obstacles=ObstacleMask(mask=mask),
    )


def make_random_env(seed: int):
    """Random world inside the dense oracle's envelope (N_c <= 64, |A| <= 16,
    N_rv <= 64, nt <= 10): (env, actions, rcfg, target)."""
    rng = np.random.default_rng(seed)
    nx = int(rng.integers(2, 9))
    ny = int(rng.integers(2, 9))
    while nx * ny > 64:
        ny = int(rng.integers(2, 9))
    nt = int(rng.integers(3, 11))
    dx = float(rng.choice([0.5, 1.0, 2.0]))
    dt = float(rng.choice([0.5, 1.0]))
    origin = (float(rng.uniform(-3.0, 3.0)), float(rng.uniform(-3.0, 3.0)))
    grid = GridSpec(nx=nx, ny=ny, nt=nt, dx=dx, dt=dt, origin=origin)
    n_modes = int(rng.integers(0, 4))
    n_real = int(rng.choice([4, 8, 16, 32, 64]))
    mean = rng.normal(0.0, 0.3 * dx / dt, size=(nt, ny, nx, 2))
    modes = rng.normal(0.0, 1.0, size=(n_modes, nt, ny, nx, 2))
    coeffs = rng.normal(0.0, 0.2 * dx / dt, size=(nt, n_real, n_modes))
    scalar = rng.uniform(0.0, 2.0, size=(nt, ny, nx))
    mask = rng.random(size=(nt, ny, nx)) < 0.08
    env = Environment(grid=grid, field=DOVelocityField(mean=mean, modes=modes, coeffs=coeffs),
                      scalar=ScalarMeanField(g_mean=scalar), obstacles=ObstacleMask(mask=mask))
    n_h, n_s = [(4, 1), (4, 2), (8, 1), (8, 2), (16, 1)][int(rng.integers(0, 5))]
    actions = ActionSpace(n_headings=n_h, n_speeds=n_s, f_max=float(rng.choice([0.5, 1.0, 1.5])) * dx / dt)
    objective = OBJECTIVES[int(rng.integers(0, len(OBJECTIVES)))]
    rcfg = RewardConfig(objective=objective, c_f=1.0, c_r=0.8, r_term=50.0, r_outbound=-200.0)
    target = (int(rng.integers(0, nx)), int(rng.integers(0, ny)))
    return env, actions, rcfg, target


def make_named_env(name: str):
    """(env, actions, rcfg, target, start) for a named workload."""
    w = workloads.get(name)
    return w.environment(), w.actions(), w.reward_config(), w.target, w.start


RANDOM_SEEDS = list(range(7000, 7020)) + [101, 301, 302, 303, 310, 320, 330] + list(range(401, 417)) + \
    [8101, 8102, 8103, 8104]


@pytest.fixture(scope="session")
def golden():
    from golden_util import load_golden
    return load_golden()


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
