"""End-to-end planner: sub-grid sizing -> model build -> backward solve, all
in HBM.  This is the path BASELINE.json's metric times:
the reference's compute_subgrid + build_model + value_iteration
(pipeline.py:96-136) without the file round trips.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .builder import DeviceEnv, build_device_model
from .core_types import PolicyValue, SubGridSpec
from .solver import solve_backward


@dataclass
class Plan:
    subgrid: SubGridSpec
    model: object        # builder.DeviceModel
    values: object       # torch f64 [N_g + 1] (device)
    policy: object       # torch int16 (u16 bits) [N_g] (device)

    def policy_value(self) -> PolicyValue:
        """Host copy in the reference's PolicyValue shape.  The backward sweep
        is exact in one pass; iterations_run reports the pass count (nt) --
        use solver.value_iteration for the reference's Jacobi sweep count."""
        v = self.values.cpu().numpy()
        a = self.policy.cpu().numpy().view(np.uint16).copy()
        return PolicyValue(values=v, actions=a, iterations_run=self.model.grid.nt, residual=0.0,
                           converged=True)


def plan(env, actions, rcfg, target, buffer: int = 1, device_env: DeviceEnv | None = None,
         subgrid: SubGridSpec | None = None) -> Plan:
    """Size the sub-grid (k_vmax), build the model (k_build) and solve it
    backward in time (k_solve_layer).  Inputs already resident in HBM are
    reused through ``device_env``."""
    # host inputs: the exact scan runs slab by slab under the upload
    denv = device_env if device_env is not None else DeviceEnv.from_host_scanned(env)
    sub = subgrid if subgrid is not None else denv.subgrid(actions.f_max, buffer)
    # the solve is queued behind the build; the build's census/overflow
    # check runs once both are in flight (one host round trip)
    dm = build_device_model(denv, actions, rcfg, target, sub, defer_check=True)
    values, policy = solve_backward(dm)
    if dm.check():   # capacity miss: the model was rebuilt, solve it again
        values, policy = solve_backward(dm, values, policy)
    return Plan(subgrid=sub, model=dm, values=values, policy=policy)
