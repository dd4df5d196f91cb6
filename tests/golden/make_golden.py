"""Generate tests/golden/golden.json by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package from a scratch copy of
/root/reference/pkg/src (the tree is read-only) and records, per case,
digests of the inputs, the built model, the value-iteration outputs and
the policy evaluation, plus a few scalars.  The parity tests check the
oracle (and, on the GPU box, the CUDA path) against these records.
Nothing under /root/reference is copied into the repository.
"""

from __future__ import annotations

import importlib
import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from golden_util import GOLDEN_JSON, env_digest, model_digest, rows_digest, sha  # noqa: E402

REF = "/root/reference/pkg"
RANDOM_SEEDS = list(range(7000, 7020)) + [101, 301, 302, 303, 310, 320, 330] + list(range(401, 417)) + \
    [8101, 8102, 8103, 8104]


def _import_reference():
    scratch = tempfile.mkdtemp(prefix="flowmdp_ref_")
    shutil.copytree(os.path.join(REF, "src"), os.path.join(scratch, "src"))
    shutil.copytree(os.path.join(REF, "tests"), os.path.join(scratch, "tests"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, os.path.join(scratch, "src"))
    sys.path.insert(0, os.path.join(scratch, "tests"))
    fm = importlib.import_module("flowmdp")
    conf = importlib.import_module("conftest")
    return fm, conf


def _solve_record(fm, model, max_iterations=None):
    from flowmdp.solver import SolverConfig, policy_value, value_iteration
    pv = value_iteration(model, SolverConfig(max_iterations=max_iterations))
    rec = {
        "values_sha": sha(pv.values), "actions_sha": sha(pv.actions),
        "iterations_run": pv.iterations_run, "residual": pv.residual, "converged": pv.converged,
    }
    if max_iterations is None:
        rec["policy_value_sha"] = sha(policy_value(model, pv.actions))
    return rec, pv


def _case(fm, env, actions, rcfg, target, n_threads=1, extra=None):
    from flowmdp.model_builder import StepContext, build_model, compute_subgrid
    ctx = StepContext(env, actions, rcfg, target)
    sub = compute_subgrid(env.field, actions, env.grid)
    model = build_model(ctx, sub, n_threads=n_threads)
    solve, pv = _solve_record(fm, model)
    rec = {
        "input_sha": env_digest(env),
        "objective": rcfg.objective,
        "target": list(target),
        "subgrid": [sub.half_width_x, sub.half_width_y],
        "nnz": model.nnz_total(),
        "model_sha": model_digest(model),
        "rewards_sha": sha(model.rewards),
        "solve": solve,
    }
    if extra:
        rec.update(extra(model, pv))
    return rec


def main():
    fm, conf = _import_reference()
    from flowmdp.environment import ActionSpace
    from flowmdp.model_builder import RewardConfig, StepContext, SubGridSpec, transition_sweep
    from flowmdp.errors import ContractViolation
    from flowmdp.synthesis import (DoubleGyreConfig, ObstacleConfig, RadiationConfig,
                                   generate_double_gyre, generate_obstacles, generate_radiation)
    from flowmdp.environment import Environment, GridSpec

    out = {"numpy": np.__version__, "random": {}, "tiny": {}, "named": {}}

    for seed in RANDOM_SEEDS:
        env, acts, rcfg, target = conf.make_random_env(seed)
        rec = _case(fm, env, acts, rcfg, target)
        rec["actions"] = [acts.n_headings, acts.n_speeds, acts.f_max]
        if seed in (413, 7001, 7013):
            rec["solve_max1"], _ = _solve_record(fm, _built(fm, env, acts, rcfg, target), max_iterations=1)
            rec["solve_max3"], _ = _solve_record(fm, _built(fm, env, acts, rcfg, target), max_iterations=3)
        out["random"][str(seed)] = rec
        print("seed", seed, rec["nnz"], rec["solve"]["iterations_run"])

    tiny = conf.make_tiny_env()
    for obj in ("time", "energy", "net_energy"):
        acts = ActionSpace(n_headings=8, n_speeds=2, f_max=1.0)
        rcfg = RewardConfig(objective=obj, c_f=1.0, c_r=0.8, r_term=50.0, r_outbound=-200.0)
        out["tiny"][obj] = _case(fm, tiny, acts, rcfg, (4, 4))

    # hand chain (test_solver.py:67-78)
    chain = conf.make_zero_flow_env(nx=3, ny=1, nt=4, dt=1.0)
    acts = ActionSpace(n_headings=1, n_speeds=1, f_max=1.0)
    rcfg = RewardConfig(objective="time", r_term=10.0, r_outbound=-50.0)
    out["chain"] = _case(fm, chain, acts, rcfg, (2, 0))

    # sub-grid violation message (test_model_builder.py:190-195)
    grid = GridSpec(nx=8, ny=4, nt=3, dx=1.0, dt=1.0)
    mean = np.zeros((3, 4, 8, 2))
    mean[..., 0] = 2.0
    from flowmdp.environment import DOVelocityField, ObstacleMask, ScalarMeanField
    venv = Environment(grid=grid, field=DOVelocityField(mean=mean, modes=np.zeros((0, 3, 4, 8, 2)),
                                                        coeffs=np.zeros((3, 3, 0))),
                       scalar=ScalarMeanField(g_mean=np.ones((3, 4, 8))),
                       obstacles=ObstacleMask(mask=np.zeros((3, 4, 8), dtype=bool)))
    vctx = StepContext(venv, ActionSpace(4, 1, 0.5), RewardConfig("time", r_term=10.0, r_outbound=-100.0), (7, 3))
    try:
        fm.build_model(vctx, SubGridSpec(1, 1))
        msg = None
    except ContractViolation as exc:
        msg = str(exc)
    out["violation_message"] = msg

    named = {
        "smoke": dict(grid=GridSpec(nx=9, ny=9, nt=10, dx=1.0, dt=0.8), amp=0.3, eps=0.15, nm=4, nr=32, seed=5,
                      rad=(1.0, 0.5, 3.0), obs=(2, 0, 0.0, ((4, 4),)), objs=("time", "energy", "net_energy"),
                      target=(6, 6), start=(2, 2)),
        "desk": dict(grid=GridSpec(nx=50, ny=50, nt=60, dx=1.0, dt=1.0), amp=0.4, eps=0.12, nm=8, nr=500, seed=42,
                     rad=(1.5, 0.5, 6.0), obs=(6, 0, 0.5, ((22, 22),)), objs=("time", "energy", "net_energy"),
                     target=(25, 38), start=(25, 12)),
    }
    for name, p in named.items():
        g = p["grid"]
        env = Environment(
            grid=g,
            field=generate_double_gyre(DoubleGyreConfig(grid=g, amplitude=p["amp"], eps=p["eps"], n_modes=p["nm"],
                                                        n_realizations=p["nr"], rng_seed=p["seed"])),
            scalar=generate_radiation(RadiationConfig(g, *p["rad"])),
            obstacles=generate_obstacles(ObstacleConfig(g, *p["obs"])),
        )
        for obj in p["objs"]:
            rcfg = RewardConfig(objective=obj, c_f=1.0, c_r=0.5, r_term=100.0, r_outbound=-300.0)
            acts = ActionSpace(n_headings=8, n_speeds=2, f_max=1.0)
            s0 = g.state_index(p["start"][0], p["start"][1], 0)

            def extra(model, pv, s0=s0):
                return {"v_start": float(pv.values[s0])}

            rec = _case(fm, env, acts, rcfg, p["target"], n_threads=os.cpu_count() or 1, extra=extra)
            out["named"][f"{name}_{obj}"] = rec
            print(name, obj, rec["nnz"], rec["solve"]["iterations_run"], rec["v_start"])

    out["pipeline"] = pipeline_records(fm)
    out["rollout"] = rollout_records(fm, conf)
    order_fixture(fm)
    os.makedirs(os.path.dirname(GOLDEN_JSON), exist_ok=True)
    with open(GOLDEN_JSON, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote", GOLDEN_JSON)


def pipeline_records(fm):
    """The reference's own file pipeline (pipeline.py:54-168): generate-env
    -> build -> solve -> rollout on pkg/configs smoke + desk x 3 objectives,
    in a scratch directory.  Records the SHA-256 of the model, policy and
    trajectory files and the rollout summary (paths dropped)."""
    import hashlib
    from flowmdp import pipeline
    from flowmdp.config import env_config_from_dict, run_config_from_dict

    def fsha(path):
        return hashlib.sha256(open(path, "rb").read()).hexdigest()

    recs = {}
    cfg_dir = os.path.join(REF, "configs")
    work = tempfile.mkdtemp(prefix="flowmdp_pipe_")
    cases = [("smoke", "smoke_env.json", "smoke_run.json", ("time", "energy", "net_energy")),
             ("desk", "desk_env.json", "desk_run_time.json", ("time", "energy", "net_energy"))]
    for name, env_file, run_file, objectives in cases:
        env_cfg = env_config_from_dict(json.load(open(os.path.join(cfg_dir, env_file))))
        env_dir = os.path.join(work, f"{name}_env")
        pipeline.run_generate_env(env_cfg, env_dir)
        base = json.load(open(os.path.join(cfg_dir, run_file)))
        for obj in objectives:
            d = dict(base)
            d.update(environment=env_dir, objective=obj, threads=os.cpu_count() or 1,
                     model=os.path.join(work, f"{name}_{obj}.model"),
                     policy=os.path.join(work, f"{name}_{obj}.policy"),
                     trajectories=os.path.join(work, f"{name}_{obj}.csv"),
                     summary=os.path.join(work, f"{name}_{obj}.summary.json"))
            cfg = run_config_from_dict(d)
            b = pipeline.run_build(cfg)
            sv = pipeline.run_solve(cfg)
            ro = pipeline.run_rollout(cfg)
            summary = {k: v for k, v in ro.items() if not k.endswith("_out")}
            recs[f"{name}_{obj}"] = {
                "run": {k: d[k] for k in ("objective", "c_f", "c_r", "r_term", "r_outbound", "n_headings",
                                          "n_speeds", "f_max", "start", "target", "epsilon")},
                "nnz_total": b["nnz_total"], "subgrid": [b["subgrid_half_width_x"], b["subgrid_half_width_y"]],
                "iterations_run": sv["iterations_run"], "residual": sv["residual"], "converged": sv["converged"],
                "model_file_sha": fsha(d["model"]), "policy_file_sha": fsha(d["policy"]),
                "trajectories_csv_sha": fsha(d["trajectories"]), "summary": summary,
            }
            print("pipeline", name, obj, b["nnz_total"], sv["iterations_run"], recs[f"{name}_{obj}"]["model_file_sha"])
    shutil.rmtree(work, ignore_errors=True)
    return recs


def rollout_records(fm, conf):
    """Reference ensemble_rollout on random worlds under the reference's VI
    policy; start = the non-target cell farthest from the target."""
    from flowmdp.model_builder import StepContext, build_model, compute_subgrid
    from flowmdp.rollout import ensemble_rollout
    from flowmdp.solver import value_iteration
    recs = {}
    for seed in RANDOM_SEEDS[:16]:
        env, acts, rcfg, target = conf.make_random_env(seed)
        ctx = StepContext(env, acts, rcfg, target)
        model = build_model(ctx, compute_subgrid(env.field, acts, env.grid))
        pv = value_iteration(model)
        g = env.grid
        start = max(((i, j) for j in range(g.ny) for i in range(g.nx) if (i, j) != tuple(target)),
                    key=lambda c: (abs(c[0] - target[0]) + abs(c[1] - target[1]), -c[1], -c[0]))
        ens = ensemble_rollout(ctx, pv.actions, start)
        recs[str(seed)] = {"start": list(start), "rows_sha": rows_digest(ens), "summary": ens.summary()}
    return recs


def order_fixture(fm):
    """Reference reduce_order on a seeded low-rank-plus-noise ensemble; the
    outputs are stored as arrays (the GPU SVD agrees to rounding, not bits)."""
    from flowmdp.synthesis import reduce_order
    rng = np.random.default_rng(2109)
    n_real, nt, ny, nx, rank = 24, 3, 5, 6, 6
    basis = rng.normal(size=(rank, nt, ny, nx, 2)) * np.linspace(3.0, 0.5, rank)[:, None, None, None, None]
    weights = rng.normal(size=(n_real, rank))
    ens = np.einsum("rk,ktyxc->rtyxc", weights, basis) + 1e-3 * rng.normal(size=(n_real, nt, ny, nx, 2)) + 0.7
    field = reduce_order(ens, 4)
    np.savez_compressed(os.path.join(os.path.dirname(GOLDEN_JSON), "reduce_order.npz"), ensemble=ens,
                        mean=field.mean, modes=field.modes, coeffs=field.coeffs)


def _built(fm, env, acts, rcfg, target):
    from flowmdp.model_builder import StepContext, build_model, compute_subgrid
    ctx = StepContext(env, acts, rcfg, target)
    return build_model(ctx, compute_subgrid(env.field, acts, env.grid))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--order-only":
        fm_, _c = _import_reference()
        order_fixture(fm_)
        print("wrote reduce_order.npz")
    elif len(sys.argv) > 1 and sys.argv[1] == "--pipeline-only":
        fm_, conf_ = _import_reference()
        gold = json.load(open(GOLDEN_JSON))
        gold["pipeline"] = pipeline_records(fm_)
        gold["rollout"] = rollout_records(fm_, conf_)
        order_fixture(fm_)
        with open(GOLDEN_JSON, "w") as fh:
            json.dump(gold, fh, indent=1, sort_keys=True)
        print("updated", GOLDEN_JSON)
    else:
        main()
