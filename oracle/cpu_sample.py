"""CPU baselines for bench.py -- TEST / MEASUREMENT INFRASTRUCTURE ONLY.

Imported by ``bench.py`` (the ``cpu_baseline`` leg of the GPU arm and the
``--impl reference`` arm), never by the product package.

Two CPU implementations of the planner step (compute_subgrid + build_model
+ value_iteration, pipeline.py:96-136) are timed on a bounded,
representative sample of the benchmarked workload:

* ``port_step``: the oracle (``flowmdp_oracle.c``, an op-for-op C
  restatement of the reference) on ALL source rows of three stratified time
  slabs t in {0, nt/3, 2nt/3}, all actions, all
  realizations, on every host core (threads over slab x row-strip jobs).
  The step = the exact sub-grid scan of those slabs + their build + value
  iteration over a model made of those slabs' rows (nt + 1 Jacobi sweeps,
  the sweep count of the reference on a full DAG model, so each sampled
  layer gets the solve work it gets in a full run).
* ``numpy_reference``: the UNMODIFIED reference package (``flowmdp``,
  installed from /root/reference/pkg into baseline/_ref) through its own
  functions -- ``compute_subgrid``, the per-slab ``_timeslice_blocks`` that
  ``build_model`` runs, its fork pool for the multi-core leg, and
  ``value_iteration`` -- on a realization-cropped sample (first R_s
  realizations; the per-transition cost does not depend on N_rv) at 1
  process and at all cores.

Rates are transitions per second over the sample's own work; a full-step
time is extrapolated from them and labelled as such.
"""

from __future__ import annotations

import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
if _HERE not in sys.path:
    sys.path.insert(0, _HERE)

import oracle as O  # noqa: E402


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            return next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "unknown CPU")
    except OSError:
        return "unknown CPU"


def stratified_slabs(nt: int, k: int = 3) -> list:
    """t in {0, nt/k, 2nt/k, ...} among the non-horizon slabs."""
    return sorted({min(nt - 2, (nt * i) // k) for i in range(k)}) if nt > 1 else [0]


class _SubField:
    """Field restricted to one slab and a row strip (contiguous copies)."""

    def __init__(self, field, t, j0, j1):
        self.mean = np.ascontiguousarray(field.mean[t:t + 1, j0:j1])
        self.modes = np.ascontiguousarray(field.modes[:, t:t + 1, j0:j1])
        self.coeffs = np.ascontiguousarray(field.coeffs[t:t + 1])


def _strips(ny: int, n: int) -> list:
    n = max(1, min(n, ny))
    cuts = [ny * k // n for k in range(n + 1)]
    return [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if a < b]


def _vi_submodel(parts, slabs, nc, n_actions):
    """Model made of the sampled slabs' rows with local state indices (slab
    k's cells at k*nc + c; columns folded onto the same local layer, SINK
    last) -- a model whose Jacobi sweeps cost what those layers cost in a
    full run.  parts[(k, strip)] = OracleModel of slab slabs[k], strip."""
    n_loc = len(slabs) * nc
    blocks = [[None] * len(slabs) for _ in range(n_actions)]
    rewards = np.zeros(n_actions * n_loc)
    for k, t in enumerate(slabs):
        mine = sorted((s, m) for (kk, s), m in parts.items() if kk == k)
        n_g = mine[0][1].n_states - 1
        for a in range(n_actions):
            rows = np.concatenate([m.blocks[a][t][0] for _, m in mine]).astype(np.int64)
            cols = np.concatenate([m.blocks[a][t][1] for _, m in mine]).astype(np.int64)
            vals = np.concatenate([m.blocks[a][t][2] for _, m in mine])
            lr = rows - t * nc + k * nc
            lc = np.where(cols == n_g, n_loc, (cols % nc) + k * nc)
            blocks[a][k] = (lr.astype(np.uint32), lc.astype(np.uint32), vals)
            for (j0, j1), m in mine:
                lo = a * n_g + t * nc
                seg = m.rewards[lo: lo + nc]
                rewards[a * n_loc + k * nc: a * n_loc + (k + 1) * nc] += seg   # zero outside the strip
    return O.OracleModel(blocks=blocks, rewards=rewards, n_states=n_loc + 1, n_actions=n_actions, nt=len(slabs))


def port_step(w, env, threads: int, slabs: list | None = None, subgrid: tuple | None = None) -> dict:
    """One sampled planner step on the oracle.  Returns timings and units."""
    g = w.grid
    slabs = slabs if slabs is not None else stratified_slabs(g.nt)
    acts, rcfg = w.actions(), w.reward_config()
    n_strips = max(1, math.ceil(threads / len(slabs)))
    jobs = [(k, s) for k in range(len(slabs)) for s in _strips(g.ny, n_strips)]
    pool = ThreadPoolExecutor(max(1, min(threads, len(jobs))))
    try:
        # compute_subgrid's exact scan over the sampled slabs (mb:392-396)
        t0 = time.perf_counter()
        mx = list(pool.map(lambda job: O.velocity_max(_SubField(env.field, slabs[job[0]], *job[1])), jobs))
        t_scan = time.perf_counter() - t0
        vx = max(m[0] for m in mx)
        vy = max(m[1] for m in mx)
        if subgrid is None:   # the sample's own maxima
            hx = int(math.ceil((vx + acts.f_max) * g.dt / g.dx)) + w.buffer
            hy = int(math.ceil((vy + acts.f_max) * g.dt / g.dx)) + w.buffer
        else:                 # the full field's (what the full build uses)
            hx, hy = subgrid
        # build: every row of the sampled slabs (mb:532-580)
        t0 = time.perf_counter()
        built = list(pool.map(
            lambda job: O.build_model(env, acts, rcfg, w.target, hx, hy, n_threads=1,
                                      t_range=(slabs[job[0]], slabs[job[0]] + 1), j_range=job[1]), jobs))
        t_build = time.perf_counter() - t0
    finally:
        pool.shutdown()
    parts = {job: m for job, m in zip(jobs, built)}
    sub = _vi_submodel(parts, slabs, g.nx * g.ny, w.n_actions)
    # value iteration (solver.py:75-109): nt + 1 Jacobi sweeps over the
    # sampled layers (the folded columns never converge, so every sweep runs)
    t0 = time.perf_counter()
    O.value_iteration(sub, epsilon=1e-300, max_iterations=g.nt + 1)
    t_vi = time.perf_counter() - t0
    units = len(slabs) * g.nx * g.ny * w.n_actions * w.n_realizations
    total = t_scan + t_build + t_vi
    return {"units": units, "seconds": total, "scan_s": t_scan, "build_s": t_build, "vi_s": t_vi,
            "slabs": slabs, "threads": min(threads, len(jobs)), "subgrid": (hx, hy),
            "full_step_s_extrapolated": total * (g.nt / len(slabs))}


def port_description(r: dict, w) -> str:
    g = w.grid
    return (f"[{cpu_model()}, os.cpu_count()={os.cpu_count()}] oracle (C restatement of the reference, -O2, no "
            f"FMA) on {w.name}: every source row of slabs t={r['slabs']} (stratified, BASELINE.md 3), "
            f"{w.n_actions} actions x {w.n_realizations} realizations = {r['units']:.3e} transitions; step = "
            f"exact sub-grid scan of those slabs ({r['scan_s']:.2f}s) + build ({r['build_s']:.2f}s) + value "
            f"iteration over those layers' rows, nt+1={g.nt + 1} Jacobi sweeps ({r['vi_s']:.2f}s) on "
            f"{r['threads']} threads (scan/build; VI single-threaded like numpy's)")


# ---------------------------------------------------------------------------
# the unmodified numpy reference (baseline/_ref)
# ---------------------------------------------------------------------------

def _ref_import(root: str):
    ref = os.path.join(root, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "flowmdp")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import flowmdp  # noqa: F401
        from flowmdp import environment, model_builder, solver
        return environment, model_builder, solver
    except Exception:
        return None


_REF_CTX = None


def _ref_worker(t):
    mb = sys.modules["flowmdp.model_builder"]
    ctx, sub = _REF_CTX
    t0 = time.perf_counter()
    blocks, rewards = mb._timeslice_blocks(ctx, sub, t)
    return t, time.perf_counter() - t0, [(b.rows, b.cols, b.vals, b.nnz) for b in blocks], rewards


def numpy_reference(w, env, root: str, r_sample: int = 200, procs: int | None = None) -> dict | None:
    """Time the unmodified reference on a realization-cropped sample: at 1
    process one stratified slab (nt/2), at all cores one slab per worker
    (stratified over the non-horizon slabs), through the reference's own
    functions and its fork pool.  None when baseline/_ref is absent."""
    mods = _ref_import(root)
    if mods is None:
        return None
    renv, mb, sol = mods
    import multiprocessing
    from concurrent.futures import ProcessPoolExecutor

    g = w.grid
    r_s = min(r_sample, w.n_realizations)
    rgrid = renv.GridSpec(nx=g.nx, ny=g.ny, nt=g.nt, dx=g.dx, dt=g.dt, origin=tuple(g.origin))
    field = renv.DOVelocityField(mean=env.field.mean, modes=env.field.modes,
                                 coeffs=np.ascontiguousarray(env.field.coeffs[:, :r_s]))
    renv_obj = renv.Environment(grid=rgrid, field=field, scalar=renv.ScalarMeanField(g_mean=env.scalar.g_mean),
                                obstacles=renv.ObstacleMask(mask=env.obstacles.mask))
    acts = renv.ActionSpace(n_headings=w.n_headings, n_speeds=w.n_speeds, f_max=w.f_max)
    rc = w.reward_config()
    rcfg = mb.RewardConfig(objective=rc.objective, c_f=rc.c_f, c_r=rc.c_r, r_term=rc.r_term,
                           r_outbound=rc.r_outbound)
    ctx = mb.StepContext(renv_obj, acts, rcfg, tuple(w.target))
    per_slab_units = g.nx * g.ny * w.n_actions * r_s
    out = {"realizations_sampled": r_s}

    # compute_subgrid on the sampled slab's field (the scan is per slab)
    t_mid = g.nt // 2
    sub_field = renv.DOVelocityField(mean=env.field.mean[t_mid:t_mid + 1], modes=env.field.modes[:, t_mid:t_mid + 1],
                                     coeffs=field.coeffs[t_mid:t_mid + 1])
    sgrid = renv.GridSpec(nx=g.nx, ny=g.ny, nt=1, dx=g.dx, dt=g.dt, origin=tuple(g.origin))
    t0 = time.perf_counter()
    mb.compute_subgrid(sub_field, acts, sgrid, buffer=w.buffer)
    t_scan = time.perf_counter() - t0
    # the build uses the full field's sub-grid (as the full run would)
    sub = mb.SubGridSpec(half_width_x=w.subgrid_hint[0], half_width_y=w.subgrid_hint[1]) if w.subgrid_hint \
        else mb.compute_subgrid(renv.DOVelocityField(mean=env.field.mean, modes=env.field.modes,
                                                     coeffs=field.coeffs), acts, rgrid, buffer=w.buffer)
    t0 = time.perf_counter()
    blocks, rewards = mb._timeslice_blocks(ctx, sub, t_mid)
    t_build = time.perf_counter() - t0
    # value iteration of that layer, nt + 1 sweeps (a one-layer model whose
    # columns fold onto the layer: it never converges early)
    nc = g.nx * g.ny
    n_g = g.nt * nc
    lb = []
    for a in range(w.n_actions):
        b = blocks[a]
        cols = np.where(b.cols.astype(np.int64) == n_g, nc, b.cols.astype(np.int64) % nc).astype(np.uint32)
        lb.append([mb.CooBlock(rows=(b.rows.astype(np.int64) - t_mid * nc).astype(np.uint32), cols=cols,
                               vals=b.vals, nnz=b.nnz)])
    model = mb.SparseModel(blocks=lb, rewards=np.ascontiguousarray(rewards.reshape(-1)), n_states=nc + 1,
                           n_actions=w.n_actions, nt=1)
    t0 = time.perf_counter()
    sol.value_iteration(model, sol.SolverConfig(epsilon=1e-300, max_iterations=g.nt + 1))
    t_vi = time.perf_counter() - t0
    # per-transition cost: the scan and the build scale with the realizations
    # sampled, value iteration does not (its work is per model entry, and a
    # row's entries barely depend on N_rv): weigh each by its own unit count
    units_full = g.nx * g.ny * w.n_actions * w.n_realizations
    per_unit = (t_scan + t_build) / per_slab_units + t_vi / units_full
    out["one_process"] = {"value": 1.0 / per_unit, "scan_s": t_scan, "build_s": t_build, "vi_s": t_vi,
                          "slab": t_mid, "units": per_slab_units,
                          "full_step_s_extrapolated": per_unit * w.transitions}
    # all cores: the reference's own fork pool, one stratified slab per worker
    procs = procs or os.cpu_count() or 1
    slabs = stratified_slabs(g.nt, min(procs, g.nt - 1))
    global _REF_CTX
    _REF_CTX = (ctx, sub)
    mp_ctx = multiprocessing.get_context("fork")
    with ProcessPoolExecutor(max_workers=len(slabs), mp_context=mp_ctx) as pool:
        list(pool.map(_ref_worker, slabs[:1]))   # fork the workers before timing
        t0 = time.perf_counter()
        res = list(pool.map(_ref_worker, slabs))
        wall = time.perf_counter() - t0
    _REF_CTX = None
    # the reference's compute_subgrid and value_iteration are single-process
    # loops over slabs / layers; only the build runs in the pool
    per_unit_all = wall / (per_slab_units * len(slabs)) + t_scan / per_slab_units + t_vi / units_full
    out["all_cores"] = {"value": 1.0 / per_unit_all, "processes": len(slabs), "slabs": slabs,
                        "build_wall_s": wall, "slab_build_s_median": float(np.median([r[1] for r in res])),
                        "full_step_s_extrapolated": per_unit_all * w.transitions}
    out["description"] = (
        f"unmodified reference (flowmdp from /root/reference/pkg, installed in baseline/_ref) on {w.name} with the "
        f"first {r_s} of {w.n_realizations} realizations (per-transition cost is independent of N_rv): 1 process = "
        f"compute_subgrid of slab {t_mid} + model_builder._timeslice_blocks(t={t_mid}) (what build_model runs per "
        f"slab) + value_iteration of that layer for nt+1 sweeps (scan and build costs per sampled transition, "
        f"VI cost per full-slab transition); all cores = the reference's fork pool building {len(slabs)} "
        f"stratified slabs (one per worker) + the single-process scan and VI shares")
    return out
