"""Stage-file formats (paper_2109_00857_b200/io.py) against the reference's
own pipeline artifacts (tests/golden: SHA-256 of the model / policy files
that pkg/src/flowmdp/pipeline.py writes for pkg/configs smoke).  CPU only:
the model comes from the oracle (C restatement) on the f32-rounded
environment the container round trip hands to the build."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle as O
from paper_2109_00857_b200 import io, workloads
from paper_2109_00857_b200.core_types import ActionSpace, CooBlock, RewardConfig, SparseModel


def _sparse(om) -> SparseModel:
    blocks = [[CooBlock(rows=r, cols=c, vals=v, nnz=int(r.size)) for (r, c, v) in row] for row in om.blocks]
    return SparseModel(blocks=blocks, rewards=om.rewards, n_states=om.n_states, n_actions=om.n_actions, nt=om.nt)


@pytest.mark.parametrize("objective", ["time", "energy", "net_energy"])
def test_smoke_model_and_policy_files_match_reference(golden, tmp_path, objective):
    rec = golden["pipeline"][f"smoke_{objective}"]
    run = rec["run"]
    w = workloads.get("smoke")
    env = io.f32_round_trip(w.environment())
    acts = ActionSpace(run["n_headings"], run["n_speeds"], run["f_max"])
    rcfg = RewardConfig(objective, c_f=run["c_f"], c_r=run["c_r"], r_term=run["r_term"],
                        r_outbound=run["r_outbound"])
    hx, hy = O.compute_subgrid(env.field, acts.f_max, env.grid)
    assert [hx, hy] == rec["subgrid"]
    om = O.build_model(env, acts, rcfg, tuple(run["target"]), hx, hy)
    assert om.nnz_total() == rec["nnz_total"]
    io.write_model(tmp_path / "m.model", _sparse(om))
    assert hashlib.sha256((tmp_path / "m.model").read_bytes()).hexdigest() == rec["model_file_sha"]

    back = io.read_model(tmp_path / "m.model")   # f32 probabilities / rewards widened, as run_solve sees them
    assert io.model_file_bytes(back) == (tmp_path / "m.model").read_bytes()
    om32 = O.OracleModel(blocks=[[(b.rows, b.cols, b.vals) for b in row] for row in back.blocks],
                         rewards=back.rewards, n_states=back.n_states, n_actions=back.n_actions, nt=back.nt)
    v, a, it, res, conv = O.value_iteration(om32, epsilon=run["epsilon"])
    assert (it, res, conv) == (rec["iterations_run"], rec["residual"], rec["converged"])
    io.write_policy(tmp_path / "p.policy", v, a)
    assert hashlib.sha256((tmp_path / "p.policy").read_bytes()).hexdigest() == rec["policy_file_sha"]
    v2, a2 = io.read_policy(tmp_path / "p.policy")
    assert np.array_equal(a2, a) and np.array_equal(v2, v.astype(np.float32).astype(np.float64))


def test_environment_container_round_trip(tmp_path):
    env = workloads.get("smoke").environment()
    io.write_environment(tmp_path / "env", env)
    back = io.read_environment(tmp_path / "env")
    ref = io.f32_round_trip(env)
    for a, b in ((back.field.mean, ref.field.mean), (back.field.modes, ref.field.modes),
                 (back.field.coeffs, ref.field.coeffs), (back.scalar.g_mean, ref.scalar.g_mean),
                 (back.obstacles.mask, ref.obstacles.mask)):
        assert a.dtype == b.dtype and np.array_equal(a, b)
    assert back.grid == env.grid


def test_bad_files_raise(tmp_path):
    from paper_2109_00857_b200.errors import InputOutputError
    (tmp_path / "x").write_bytes(b"NOTAMODEL" + bytes(40))
    with pytest.raises(InputOutputError):
        io.read_model(tmp_path / "x")
    with pytest.raises(InputOutputError):
        io.read_policy(tmp_path / "x")
    with pytest.raises(InputOutputError):
        io.write_policy(tmp_path / "p", np.zeros(5), np.zeros(3, dtype=np.uint16))
