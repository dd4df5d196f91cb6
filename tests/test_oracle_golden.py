"""Pin the CPU oracle (oracle/flowmdp_oracle.c) to the reference's own
outputs (tests/golden/golden.json, written by make_golden.py from the
unmodified reference).  CPU only."""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle as O
from conftest import RANDOM_SEEDS, make_named_env, make_random_env, make_tiny_env, make_zero_flow_env
from golden_util import env_digest, model_digest, sha
from paper_2109_00857_b200.core_types import ActionSpace, RewardConfig


def _check_case(rec, env, acts, rcfg, target, n_threads=1):
    assert env_digest(env) == rec["input_sha"], "input generator drifted from the reference"
    hx, hy = O.compute_subgrid(env.field, acts.f_max, env.grid)
    assert [hx, hy] == rec["subgrid"]
    model = O.build_model(env, acts, rcfg, target, hx, hy, n_threads=n_threads)
    assert model.nnz_total() == rec["nnz"]
    assert sha(model.rewards) == rec["rewards_sha"]
    assert model_digest(model) == rec["model_sha"]
    values, actions, iters, res, conv = O.value_iteration(model)
    s = rec["solve"]
    assert sha(values) == s["values_sha"]
    assert sha(actions) == s["actions_sha"]
    assert (iters, res, conv) == (s["iterations_run"], s["residual"], s["converged"])
    assert sha(O.policy_value(model, actions)) == s["policy_value_sha"]
    return model, values, actions


@pytest.mark.parametrize("seed", RANDOM_SEEDS)
def test_oracle_random_env(golden, seed):
    rec = golden["random"][str(seed)]
    env, acts, rcfg, target = make_random_env(seed)
    model, values, _ = _check_case(rec, env, acts, rcfg, target)
    for key, mi in (("solve_max1", 1), ("solve_max3", 3)):
        if key in rec:
            v, a, it, res, conv = O.value_iteration(model, max_iterations=mi)
            assert sha(v) == rec[key]["values_sha"] and sha(a) == rec[key]["actions_sha"]
            assert (it, res, conv) == (rec[key]["iterations_run"], rec[key]["residual"], rec[key]["converged"])


@pytest.mark.parametrize("objective", ["time", "energy", "net_energy"])
def test_oracle_tiny_env(golden, objective):
    acts = ActionSpace(n_headings=8, n_speeds=2, f_max=1.0)
    rcfg = RewardConfig(objective=objective, c_f=1.0, c_r=0.8, r_term=50.0, r_outbound=-200.0)
    _check_case(golden["tiny"][objective], make_tiny_env(), acts, rcfg, (4, 4))


def test_oracle_hand_chain(golden):
    env = make_zero_flow_env(nx=3, ny=1, nt=4, dt=1.0)
    acts = ActionSpace(n_headings=1, n_speeds=1, f_max=1.0)
    rcfg = RewardConfig(objective="time", r_term=10.0, r_outbound=-50.0)
    _, values, _ = _check_case(golden["chain"], env, acts, rcfg, (2, 0))
    assert values[0] == 8.0 and values[1] == 9.0 and values[env.grid.sink] == 0.0


def test_oracle_violation_message(golden):
    from paper_2109_00857_b200.core_types import DOVelocityField, Environment, GridSpec, ObstacleMask, \
        ScalarMeanField
    grid = GridSpec(nx=8, ny=4, nt=3, dx=1.0, dt=1.0)
    mean = np.zeros((3, 4, 8, 2))
    mean[..., 0] = 2.0
    env = Environment(grid=grid, field=DOVelocityField(mean, np.zeros((0, 3, 4, 8, 2)), np.zeros((3, 3, 0))),
                      scalar=ScalarMeanField(np.ones((3, 4, 8))),
                      obstacles=ObstacleMask(np.zeros((3, 4, 8), dtype=bool)))
    with pytest.raises(O.OracleViolation) as ei:
        O.build_model(env, ActionSpace(4, 1, 0.5), RewardConfig("time", r_term=10.0, r_outbound=-100.0),
                      (7, 3), 1, 1)
    assert str(ei.value) == golden["violation_message"]


@pytest.mark.parametrize("objective", ["time", "energy", "net_energy"])
def test_oracle_smoke(golden, objective):
    env, acts, rcfg, target, start = make_named_env("smoke")
    rcfg = RewardConfig(objective, c_f=1.0, c_r=0.5, r_term=100.0, r_outbound=-300.0)
    rec = golden["named"][f"smoke_{objective}"]
    _, values, _ = _check_case(rec, env, acts, rcfg, target)
    assert values[env.grid.state_index(*start, 0)] == rec["v_start"]


@pytest.mark.parametrize("objective", ["time", "energy", "net_energy"])
def test_oracle_desk(golden, objective):
    """Desk C1 (50x50x60, 16 actions, 500 realizations): ~1.2e9 transitions."""
    env, acts, rcfg, target, start = make_named_env("desk")
    rcfg = RewardConfig(objective, c_f=1.0, c_r=0.5, r_term=100.0, r_outbound=-300.0)
    rec = golden["named"][f"desk_{objective}"]
    _, values, _ = _check_case(rec, env, acts, rcfg, target, n_threads=os.cpu_count() or 1)
    assert values[env.grid.state_index(*start, 0)] == rec["v_start"]


def test_oracle_thread_invariance():
    env, acts, rcfg, target = make_random_env(320)
    hx, hy = O.compute_subgrid(env.field, acts.f_max, env.grid)
    one = O.build_model(env, acts, rcfg, target, hx, hy, n_threads=1)
    many = O.build_model(env, acts, rcfg, target, hx, hy, n_threads=4)
    assert model_digest(one) == model_digest(many)
