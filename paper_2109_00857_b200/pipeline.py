"""File-to-file planner stages on the B200 path (the reference's
pipeline.run_build / run_solve / run_rollout, pipeline.py:96-168).

These are the callers of the hot path: they read the reference's stage
files, run the CUDA build / solve / rollout and write byte-identical stage
files.  ``cfg`` is a mapping with the reference's run-config keys
(environment, model, policy, trajectories, summary, objective, c_f, c_r,
r_term, r_outbound, n_headings, n_speeds, f_max, start, target, epsilon,
max_iterations, subgrid_buffer); JSON parsing / CLI / service stay out of
scope.
"""

from __future__ import annotations

import time

from . import io
from .builder import build_device_model, compute_subgrid
from .core_types import ActionSpace, RewardConfig, SolverConfig, StepContext
from .errors import ContractViolation
from .rollout import ensemble_rollout
from .solver import value_iteration


# RunConfig defaults of the reference (config.py:182-196): a run config that
# omits a key builds the same actions and rewards as the reference pipeline
RUN_DEFAULTS = {"objective": "time", "c_f": 1.0, "c_r": 1.0, "r_term": 100.0, "r_outbound": -1000.0,
                "n_headings": 8, "n_speeds": 2, "f_max": 1.0, "epsilon": 1e-8, "max_iterations": None,
                "subgrid_buffer": 1}


def _get(cfg, key):
    v = cfg.get(key)
    return RUN_DEFAULTS[key] if v is None else v


def _actions(cfg) -> ActionSpace:
    return ActionSpace(n_headings=int(_get(cfg, "n_headings")), n_speeds=int(_get(cfg, "n_speeds")),
                       f_max=float(_get(cfg, "f_max")))


def _rewards(cfg) -> RewardConfig:
    return RewardConfig(objective=_get(cfg, "objective"), c_f=float(_get(cfg, "c_f")),
                        c_r=float(_get(cfg, "c_r")), r_term=float(_get(cfg, "r_term")),
                        r_outbound=float(_get(cfg, "r_outbound")))


def run_build(cfg) -> dict:
    """Environment container -> model file (pipeline.py:96-120)."""
    env = io.read_environment(cfg["environment"])
    acts = _actions(cfg)
    ctx = StepContext(env, acts, _rewards(cfg), tuple(cfg["target"]))
    denv = ctx.device_env()
    sub = compute_subgrid(env.field, acts, env.grid, buffer=int(_get(cfg, "subgrid_buffer")), device_env=denv)
    t0 = time.perf_counter()
    dm = build_device_model(denv, acts, ctx.rcfg, ctx.target, sub)
    elapsed = time.perf_counter() - t0
    io.write_model(cfg["model"], dm)
    return {"out": str(cfg["model"]), "n_states": dm.n_states, "n_actions": dm.n_actions, "nt": dm.nt,
            "nnz_total": dm.nnz, "subgrid_half_width_x": sub.half_width_x, "subgrid_half_width_y": sub.half_width_y,
            "build_seconds": elapsed}


def run_solve(cfg) -> dict:
    """Model file -> policy file by value iteration (pipeline.py:123-136): the
    model's f32 probabilities / rewards widened to f64, as the reference reads them."""
    model = io.read_model(cfg["model"])
    pv = value_iteration(model, SolverConfig(epsilon=float(_get(cfg, "epsilon")),
                                             max_iterations=_get(cfg, "max_iterations")))
    io.write_policy(cfg["policy"], pv.values, pv.actions)
    return {"out": str(cfg["policy"]), "iterations_run": pv.iterations_run, "residual": pv.residual,
            "converged": pv.converged}


def run_rollout(cfg) -> dict:
    """Policy file -> trajectories CSV + summary JSON (pipeline.py:139-168)."""
    env = io.read_environment(cfg["environment"])
    values, actions = io.read_policy(cfg["policy"])
    if values.shape[0] != env.grid.n_states + 1:
        raise ContractViolation("policy file does not match the environment's state count")
    start, target = tuple(cfg["start"]), tuple(cfg["target"])
    ctx = StepContext(env, _actions(cfg), _rewards(cfg), target)
    ens = ensemble_rollout(ctx, actions, start)
    io.write_trajectories_csv(cfg["trajectories"], ens)
    summary = ens.summary()
    summary.update({"objective": _get(cfg, "objective"), "start": list(start), "target": list(target),
                    "policy_value_at_start": float(values[env.grid.state_index(start[0], start[1], 0)]),
                    "trajectories_out": str(cfg["trajectories"])})
    spath = cfg.get("summary") or (str(cfg["trajectories"]) + ".summary.json")
    io.write_summary_json(spath, summary)
    summary["summary_out"] = str(spath)
    return summary


__all__ = ["run_build", "run_solve", "run_rollout"]
