"""Ensemble rollout on the B200: drop-in for the reference's rollout.py.

SURVEY.md 8(f) row 1: the consumer of the solved policy.  Every
realization's trajectory runs in its own thread of ``k_rollout``
(csrc/flowmdp_b200.cu): reconstruct_at + step_flat with causes
(model_builder.py:286-369), cumulative reward in step order, rows recorded
on the device; the host only formats them into the reference's
``Trajectory`` rows (rollout.py:50-105).  Results are bit-identical to
``ensemble_rollout`` / ``simulate_trajectory`` (rollout.py:107-208); thread
counts are accepted and ignored.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .builder import action_records
from .core_types import OBJECTIVE_CODE
from .errors import ContractViolation

CAUSE_MOVE, CAUSE_TARGET, CAUSE_OUTSIDE, CAUSE_HORIZON, CAUSE_OBSTACLE_LAND, CAUSE_OBSTACLE_TRANSIT = range(6)
STATUS_REACHED, STATUS_OUTBOUND, STATUS_HORIZON = "reached_target", "outbound", "horizon"
_STATUS_BY_CAUSE = {1: STATUS_REACHED, 2: STATUS_OUTBOUND, 3: STATUS_HORIZON, 4: STATUS_OUTBOUND,
                    5: STATUS_OUTBOUND}
QUANTILES = (0.05, 0.25, 0.5, 0.75, 0.95)


@dataclass
class Trajectory:
    """One realization's rows (step, t, x, y, action, reward, cum_reward,
    status) and outcome (rollout.py:50-72)."""

    realization: int
    status: str
    final_cause: int
    rows: list
    cum_reward: float
    n_steps: int
    arrival_t: int | None


@dataclass
class TrajectoryEnsemble:
    """Trajectories in realization order (rollout.py:75-104)."""

    trajectories: list

    def cumulative_rewards(self) -> np.ndarray:
        return np.array([tr.cum_reward for tr in self.trajectories], dtype=np.float64)

    def status_counts(self) -> dict:
        counts = {STATUS_REACHED: 0, STATUS_OUTBOUND: 0, STATUS_HORIZON: 0}
        for tr in self.trajectories:
            counts[tr.status] += 1
        return counts

    def summary(self) -> dict:
        cum = self.cumulative_rewards()
        n = cum.size
        std = float(cum.std(ddof=1)) if n > 1 else 0.0
        arr = [tr.arrival_t for tr in self.trajectories if tr.arrival_t is not None]
        return {
            "n_trajectories": n,
            "mean_cum_reward": float(cum.mean()),
            "std_cum_reward": std,
            "stderr_cum_reward": std / float(np.sqrt(n)) if n > 0 else 0.0,
            "quantiles_cum_reward": {str(q): float(v) for q, v in zip(QUANTILES, np.quantile(cum, QUANTILES))},
            "status_counts": self.status_counts(),
            "mean_arrival_t": float(np.mean(arr)) if arr else None,
            "min_arrival_t": int(min(arr)) if arr else None,
            "max_arrival_t": int(max(arr)) if arr else None,
        }


def _device_policy(policy, n_g: int, dev):
    import torch
    if isinstance(policy, torch.Tensor):
        p = policy.to(dev)
        return p if p.dtype == torch.int16 else p.to(torch.int32).to(torch.int16)
    a = np.ascontiguousarray(np.asarray(policy).astype(np.uint16)).view(np.int16)
    return torch.from_numpy(a).to(dev)


def rollout_device(ctx, policy, start, realizations):
    """Run ``k_rollout`` for the given realizations.  Returns host arrays
    (n_rows, final_cell, row_cell, row_action, row_cause, row_reward, row_cum)."""
    import torch
    grid = ctx.grid
    denv = ctx.device_env()
    dev = denv.mean.device
    recs = action_records(ctx.actions, ctx.rcfg, grid)
    d_act = denv.action_table(recs)
    d_gate = denv.gate_radius_device(float(ctx.actions.f_max))
    n = len(realizations)
    mr = grid.nt
    d_real = torch.tensor(np.asarray(realizations, dtype=np.int32), device=dev)
    pol = _device_policy(policy, grid.n_states, dev)
    out = {
        "row_cell": torch.empty(n * mr, dtype=torch.int32, device=dev),
        "row_action": torch.empty(n * mr, dtype=torch.int16, device=dev),
        "row_cause": torch.empty(n * mr, dtype=torch.int8, device=dev),
        "row_reward": torch.empty(n * mr, dtype=torch.float64, device=dev),
        "row_cum": torch.empty(n * mr, dtype=torch.float64, device=dev),
        "n_rows": torch.empty(n, dtype=torch.int32, device=dev),
        "final_cell": torch.empty(n, dtype=torch.int32, device=dev),
    }
    rcfg = ctx.rcfg
    ti, tj = ctx.target
    rw = _lib.FmReward(OBJECTIVE_CODE[rcfg.objective], float(rcfg.c_f), float(rcfg.c_r), float(rcfg.r_term),
                       float(rcfg.r_outbound), ti, tj)
    args = _lib.FmRolloutArgs(denv.fm_grid(), denv.fm_env(), rw, d_act.data_ptr(), recs.shape[0],
                              denv.sat.data_ptr(), d_gate.data_ptr(), pol.data_ptr(), int(start[0]), int(start[1]),
                              d_real.data_ptr(), n, mr, *(out[k].data_ptr() for k in (
                                  "row_cell", "row_action", "row_cause", "row_reward", "row_cum", "n_rows",
                                  "final_cell")))
    _lib.check(_lib.load().fm_rollout(C.byref(args), _lib.stream_ptr()), "fm_rollout")
    h = {k: v.cpu().numpy() for k, v in out.items()}
    shape = (n, mr)
    return (h["n_rows"], h["final_cell"], h["row_cell"].reshape(shape), h["row_action"].reshape(shape),
            h["row_cause"].reshape(shape), h["row_reward"].reshape(shape), h["row_cum"].reshape(shape))


def _trajectories(ctx, policy, start, reals) -> list:
    grid = ctx.grid
    si, sj = int(start[0]), int(start[1])
    if not (0 <= si < grid.nx and 0 <= sj < grid.ny):
        raise ContractViolation(f"start cell {tuple(start)} outside grid")
    n_act = ctx.act_vecs.shape[0]
    if np.shape(policy)[0]:
        p_min = int(policy.min()) if hasattr(policy, "min") else int(min(policy))
        p_max = int(policy.max()) if hasattr(policy, "max") else int(max(policy))
        if p_min < 0 or p_max >= n_act:
            bad = p_max if p_max >= n_act else p_min
            raise ContractViolation(f"policy action {bad} out of range")
    # realization indices follow numpy indexing of coeffs[t, r] (rollout.py:
    # reconstruct_timeslice): negatives wrap, anything else out of range raises
    n_real = int(ctx.env.field.coeffs.shape[1])
    dev_reals = []
    for r in reals:
        if not -n_real <= r < n_real:
            raise IndexError(f"index {r} is out of bounds for axis 1 with size {n_real}")
        dev_reals.append(r + n_real if r < 0 else r)
    centers = grid.cell_centers()
    cell0 = sj * grid.nx + si
    if bool(np.asarray(ctx.env.obstacles.mask)[0].reshape(-1)[cell0]):
        # start cell masked at t = 0: one outbound row (rollout.py:124-136)
        x, y = centers[cell0]
        r_out = ctx.rcfg.r_outbound
        return [Trajectory(realization=r, status=STATUS_OUTBOUND, final_cause=CAUSE_OBSTACLE_LAND,
                           rows=[(0, 0, float(x), float(y), -1, r_out, r_out, STATUS_OUTBOUND)], cum_reward=r_out,
                           n_steps=0, arrival_t=None)
                for r in reals]
    if not reals:
        return []
    n_rows, fin, rc, ra, rca, rr, rcum = rollout_device(ctx, policy, (si, sj), dev_reals)
    xs, ys = centers[:, 0].tolist(), centers[:, 1].tolist()
    trajs = []
    for k, r in enumerate(reals):
        n = int(n_rows[k])
        cells, acts, causes = rc[k, :n].tolist(), ra[k, :n].tolist(), rca[k, :n].tolist()
        rews, cums = rr[k, :n].tolist(), rcum[k, :n].tolist()
        rows = []
        for s in range(n):   # step s departs at time s (rollout.py:141-151)
            c, cause = cells[s], causes[s]
            terminal = s == n - 1 and cause != CAUSE_TARGET
            rows.append((s, s, xs[c], ys[c], acts[s], rews[s], cums[s],
                         _STATUS_BY_CAUSE[cause] if terminal else "ok"))
        cause = causes[-1]
        if cause == CAUSE_TARGET:   # arrival row at the target centre (rollout.py:152-166)
            f = int(fin[k])
            rows.append((n, n, xs[f], ys[f], -1, 0.0, cums[-1], STATUS_REACHED))
            trajs.append(Trajectory(realization=r, status=STATUS_REACHED, final_cause=cause, rows=rows,
                                    cum_reward=cums[-1], n_steps=n, arrival_t=n))
        else:
            trajs.append(Trajectory(realization=r, status=_STATUS_BY_CAUSE[cause], final_cause=cause, rows=rows,
                                    cum_reward=cums[-1], n_steps=n, arrival_t=None))
    return trajs


def ensemble_rollout(ctx, policy, start, n_threads: int = 1, realizations=None) -> TrajectoryEnsemble:
    """Drop-in for rollout.ensemble_rollout (rollout.py:180-208)."""
    del n_threads
    if np.shape(policy)[0] != ctx.grid.n_states:
        raise ContractViolation("policy length must equal the non-sink state count")
    if tuple(int(x) for x in start) == tuple(ctx.target):
        raise ContractViolation("start cell equals target cell")
    reals = list(range(ctx.env.field.coeffs.shape[1])) if realizations is None else [int(r) for r in realizations]
    return TrajectoryEnsemble(_trajectories(ctx, policy, start, reals))


def simulate_trajectory(ctx, policy, start, realization: int) -> Trajectory:
    """Drop-in for rollout.simulate_trajectory (rollout.py:107-177)."""
    return _trajectories(ctx, policy, start, [int(realization)])[0]
