"""B200-native MDP model build + value-iteration solve (arXiv 2109.00857).

Drop-in for the hot path of the reference package ``flowmdp``:

    compute_subgrid, build_model          (model_builder.py:376, :532)
    value_iteration, extract_policy,
    policy_value                          (solver.py:75, :112, :122)

with the reference's value types and errors, plus the device-resident
planner ``plan`` (build + backward solve without leaving HBM), and the
stages around it: ``ensemble_rollout`` / ``simulate_trajectory``
(rollout.py), ``reduce_order`` (synthesis.py), the stage files (``io``) and
the file pipeline (``pipeline``).  The compute
runs in hand-written sm_100a CUDA (csrc/flowmdp_b200.cu) behind the C ABI
in include/flowmdp_b200.h; there is no CPU fallback.
"""

__version__ = "0.1.0"

from .core_types import (
    OUTSIDE,
    ActionSpace,
    CooBlock,
    DOVelocityField,
    Environment,
    GridSpec,
    ObstacleMask,
    PolicyValue,
    RewardConfig,
    ScalarMeanField,
    SolverConfig,
    SparseModel,
    StepContext,
    SubGridSpec,
    storage_footprint,
)
from .errors import (
    ConfigError,
    ContractViolation,
    FlowMdpError,
    InputOutputError,
    NativeUnavailable,
    VerificationFailure,
)
from .builder import DeviceEnv, DeviceModel, build_device_model, build_model, compute_subgrid
from .solver import extract_policy, policy_value, solve_backward, value_iteration
from .planner import Plan, plan
from .order import reduce_order
from .rollout import Trajectory, TrajectoryEnsemble, ensemble_rollout, simulate_trajectory

__all__ = [
    "OUTSIDE", "ActionSpace", "CooBlock", "DOVelocityField", "Environment", "GridSpec", "ObstacleMask",
    "PolicyValue", "RewardConfig", "ScalarMeanField", "SolverConfig", "SparseModel", "StepContext",
    "SubGridSpec", "storage_footprint",
    "ConfigError", "ContractViolation", "FlowMdpError", "InputOutputError", "NativeUnavailable",
    "VerificationFailure",
    "DeviceEnv", "DeviceModel", "build_device_model", "build_model", "compute_subgrid",
    "extract_policy", "policy_value", "solve_backward", "value_iteration",
    "Plan", "plan",
    "reduce_order", "Trajectory", "TrajectoryEnsemble", "ensemble_rollout", "simulate_trajectory",
]
