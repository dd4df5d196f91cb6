"""Host-side logic that needs no GPU: run-config defaults of the file
pipeline and argument validation that must fail before any device work."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import make_named_env
from paper_2109_00857_b200 import ContractViolation, StepContext
from paper_2109_00857_b200.pipeline import _actions, _rewards


def test_run_config_defaults_are_the_reference_runconfig():
    """A run config that omits the optional keys gets the reference's
    RunConfig defaults (config.py:182-196): 8 headings x 2 speeds, f_max 1,
    c_f 1, c_r 1, r_term 100, r_outbound -1000, time objective."""
    a = _actions({})
    assert (a.n_headings, a.n_speeds, a.f_max) == (8, 2, 1.0)
    r = _rewards({})
    assert (r.objective, r.c_f, r.c_r, r.r_term, r.r_outbound) == ("time", 1.0, 1.0, 100.0, -1000.0)
    # explicit keys win; an explicit null falls back to the default
    a = _actions({"n_headings": 4, "n_speeds": None, "f_max": 0.5})
    assert (a.n_headings, a.n_speeds, a.f_max) == (4, 2, 0.5)
    r = _rewards({"objective": "energy", "c_r": 0.25})
    assert (r.objective, r.c_r, r.r_outbound) == ("energy", 0.25, -1000.0)


def _smoke_ctx():
    env, acts, rcfg, target, start = make_named_env("smoke")
    return StepContext(env, acts, rcfg, target), start


def test_rollout_rejects_out_of_range_realizations_before_launch():
    """numpy indexing of coeffs[t, r] (reference rollout): r >= N_rv and
    r < -N_rv raise IndexError -- here before any device work."""
    from paper_2109_00857_b200.rollout import ensemble_rollout
    ctx, start = _smoke_ctx()
    pol = np.zeros(ctx.grid.n_states, dtype=np.uint16)
    n_real = ctx.env.field.coeffs.shape[1]
    with pytest.raises(IndexError):
        ensemble_rollout(ctx, pol, start, realizations=[0, n_real])
    with pytest.raises(IndexError):
        ensemble_rollout(ctx, pol, start, realizations=[-n_real - 1])


def test_rollout_rejects_out_of_range_policy_entries():
    from paper_2109_00857_b200.rollout import ensemble_rollout
    ctx, start = _smoke_ctx()
    n_a = ctx.actions.n_actions
    pol = np.zeros(ctx.grid.n_states, dtype=np.int64)
    pol[3] = n_a
    with pytest.raises(ContractViolation):
        ensemble_rollout(ctx, pol, start)
    pol[3] = -1
    with pytest.raises(ContractViolation):
        ensemble_rollout(ctx, pol, start)
