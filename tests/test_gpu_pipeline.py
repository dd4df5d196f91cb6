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
