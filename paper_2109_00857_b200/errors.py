"""Error taxonomy of the drop-in boundary.

Same class names, categories and exit codes as the reference package
(/root/reference/pkg/src/flowmdp/errors.py:8-58) so callers that branch on
``ContractViolation`` or on ``exit_code`` keep working.
"""

EXIT_OK, EXIT_CONFIG, EXIT_IO, EXIT_CONTRACT, EXIT_VERIFY = 0, 2, 3, 4, 5


class FlowMdpError(Exception):
    exit_code = 1
    category = "error"


class ConfigError(FlowMdpError):
    exit_code = EXIT_CONFIG
    category = "config"


class InputOutputError(FlowMdpError):
    exit_code = EXIT_IO
    category = "io"


class ContractViolation(FlowMdpError):
    """Broken precondition (bad index, undersized sub-grid, shape mismatch).
    Never swallowed; always aborts the operation."""

    exit_code = EXIT_CONTRACT
    category = "contract"


class VerificationFailure(FlowMdpError):
    exit_code = EXIT_VERIFY
    category = "verification"


class NativeUnavailable(RuntimeError):
    """The sm_100a extension is missing or no CUDA device is present.

    There is deliberately no CPU fallback on the product path."""
