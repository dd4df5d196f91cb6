"""The rows SURVEY.md 8(f) ranks next, on the GPU, against the reference's
own artifacts (tests/golden, made by tests/golden/make_golden.py):

  * pipeline: environment container -> CUDA build -> model file (device
    image) -> value iteration -> policy file -> CUDA rollout -> trajectory
    CSV + summary, byte-identical to pkg/src/flowmdp/pipeline.py on the
    pkg/configs smoke and desk missions, three objectives each;
  * ensemble_rollout on random worlds under the value-iteration policy;
  * the device model image equals the host writer's bytes."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import make_random_env
from golden_util import rows_digest

pytestmark = pytest.mark.gpu

fm = pytest.importorskip("paper_2109_00857_b200")
from paper_2109_00857_b200 import io, pipeline, workloads  # noqa: E402
from paper_2109_00857_b200.rollout import ensemble_rollout, simulate_trajectory  # noqa: E402


def _fsha(p) -> str:
    return hashlib.sha256(open(p, "rb").read()).hexdigest()


@pytest.mark.parametrize("case", ["smoke_time", "smoke_energy", "smoke_net_energy",
                                  "desk_time", "desk_energy", "desk_net_energy"])
def test_pipeline_artifacts_match_reference(golden, tmp_path, case):
    rec = golden["pipeline"][case]
    name = case.split("_")[0]
    io.write_environment(tmp_path / "env", workloads.get(name).environment())
    cfg = dict(rec["run"], environment=str(tmp_path / "env"), model=str(tmp_path / "m.model"),
               policy=str(tmp_path / "p.policy"), trajectories=str(tmp_path / "t.csv"),
               summary=str(tmp_path / "s.json"), subgrid_buffer=1)
    b = pipeline.run_build(cfg)
    assert b["nnz_total"] == rec["nnz_total"]
    assert [b["subgrid_half_width_x"], b["subgrid_half_width_y"]] == rec["subgrid"]
    assert _fsha(cfg["model"]) == rec["model_file_sha"]
    s = pipeline.run_solve(cfg)
    assert (s["iterations_run"], s["residual"], s["converged"]) == (rec["iterations_run"], rec["residual"],
                                                                    rec["converged"])
    assert _fsha(cfg["policy"]) == rec["policy_file_sha"]
    r = pipeline.run_rollout(cfg)
    assert _fsha(cfg["trajectories"]) == rec["trajectories_csv_sha"]
    assert {k: v for k, v in r.items() if not k.endswith("_out")} == rec["summary"]


@pytest.mark.parametrize("seed", [7000, 7001, 7002, 7003, 7004, 7005, 7006, 7007, 7008, 7009, 7010, 7011, 7012,
                                  7013, 7014, 7015])
def test_rollout_random_worlds(golden, seed):
    rec = golden["rollout"][str(seed)]
    env, acts, rcfg, target = make_random_env(seed)
    ctx = fm.StepContext(env, acts, rcfg, target)
    model = fm.build_model(ctx, fm.compute_subgrid(env.field, acts, env.grid))
    pv = fm.value_iteration(model)
    ens = ensemble_rollout(ctx, pv.actions, tuple(rec["start"]))
    assert rows_digest(ens) == rec["rows_sha"]
    assert ens.summary() == rec["summary"]
    one = simulate_trajectory(ctx, pv.actions, tuple(rec["start"]), 3 % env.field.coeffs.shape[1])
    assert one == ens.trajectories[3 % env.field.coeffs.shape[1]]


def test_device_model_image_equals_host_writer():
    env, acts, rcfg, target = make_random_env(7002)
    ctx = fm.StepContext(env, acts, rcfg, target)
    sub = fm.compute_subgrid(env.field, acts, env.grid)
    dm = fm.build_device_model(ctx.device_env(), acts, rcfg, target, sub)
    assert io.model_file_bytes(dm) == io.model_file_bytes(dm.to_sparse_model())


def test_rollout_contract_errors():
    env, acts, rcfg, target = make_random_env(7003)
    ctx = fm.StepContext(env, acts, rcfg, target)
    pol = np.zeros(env.grid.n_states, dtype=np.uint16)
    with pytest.raises(fm.ContractViolation):
        ensemble_rollout(ctx, pol[:-1], (0, 0) if tuple(target) != (0, 0) else (1, 0))
    with pytest.raises(fm.ContractViolation):
        ensemble_rollout(ctx, pol, tuple(target))


def test_rollout_negative_realizations_wrap_like_numpy():
    """coeffs[t, r] with r < 0 wraps (numpy indexing in the reference's
    rollout): trajectory -1 follows realization N_rv - 1 and keeps -1 as
    its label."""
    env, acts, rcfg, target = make_random_env(7001)
    ctx = fm.StepContext(env, acts, rcfg, target)
    pv = fm.value_iteration(fm.build_model(ctx, fm.compute_subgrid(env.field, acts, env.grid)))
    start = (0, 0) if tuple(target) != (0, 0) else (1, 0)
    n_real = env.field.coeffs.shape[1]
    a = simulate_trajectory(ctx, pv.actions, start, -1)
    b = simulate_trajectory(ctx, pv.actions, start, n_real - 1)
    assert a.realization == -1 and b.realization == n_real - 1
    assert a.rows == b.rows and a.status == b.status and a.cum_reward == b.cum_reward


def test_export_of_a_deferred_build_runs_the_check_first():
    """to_sparse_model / value_iteration on a model built with defer_check
    (and an entry buffer too small for it) finish the census / capacity
    retry before sizing the export: same model as the checked build."""
    env, acts, rcfg, target = make_random_env(7004)
    ctx = fm.StepContext(env, acts, rcfg, target)
    sub = fm.compute_subgrid(env.field, acts, env.grid)
    denv = ctx.device_env()
    ref = fm.build_device_model(denv, acts, rcfg, target, sub).to_sparse_model()
    dm = fm.build_device_model(denv, acts, rcfg, target, sub, defer_check=True, capacity_hint=1)
    sm = dm.to_sparse_model()
    assert sm.nnz_total() == ref.nnz_total()
    for a in range(acts.n_actions):
        for t in range(env.grid.nt):
            x, y = sm.blocks[a][t], ref.blocks[a][t]
            assert np.array_equal(x.rows, y.rows) and np.array_equal(x.cols, y.cols)
            assert x.vals.tobytes() == y.vals.tobytes()
    assert sm.rewards.tobytes() == ref.rewards.tobytes()
    dm2 = fm.build_device_model(denv, acts, rcfg, target, sub, defer_check=True, capacity_hint=1)
    pv = fm.value_iteration(dm2)
    pv_ref = fm.value_iteration(ref)
    assert pv.values.tobytes() == pv_ref.values.tobytes()
