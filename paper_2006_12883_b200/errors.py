"""Exception types of the drop-in API (mirrors paradiff/errors.py:4-9).

Status codes coming back from the C-ABI (`include/paradiff_b200.h`) map onto
these: PD_ERR_CONFIG -> ConfigurationError, PD_ERR_SOLVER -> SolverError,
PD_ERR_CUDA -> DeviceError (a SolverError subclass, so reference callers that
catch SolverError keep working).
"""


class ConfigurationError(ValueError):
    """Invalid discretization or solver configuration (bad sizes, unknown kinds)."""


class SolverError(RuntimeError):
    """Numerical failure inside a solver (zero pivot, NaN, singular system)."""


class DeviceError(SolverError):
    """CUDA runtime failure inside the native library."""
