"""Exception types mirroring the reference's (errors.hpp:10-47)."""
from __future__ import annotations

from . import abi


class IgnisError(RuntimeError):
    status = abi.IGN_INTERNAL_ERROR


class ConfigError(IgnisError):
    status = abi.IGN_CONFIG_ERROR


class StateError(IgnisError):
    status = abi.IGN_STATE_ERROR


class NumericsError(IgnisError):
    status = abi.IGN_NUMERICS_ERROR


class StepFailure(NumericsError):
    """errors.hpp:29-35: a step produced an invalid state at (stage, i, j)."""
    status = abi.IGN_STEP_FAILURE

    def __init__(self, what: str, stage: int, i: int, j: int, k: int = 0):
        super().__init__(what)
        self.stage, self.i, self.j, self.k = stage, i, j, k  # k: 3D extension


class FormatError(IgnisError):
    status = abi.IGN_FORMAT_ERROR


class UsageError(IgnisError):
    status = abi.IGN_USAGE_ERROR


class CudaError(IgnisError):
    status = abi.IGN_CUDA_ERROR


_BY_STATUS = {c.status: c for c in
              (ConfigError, StateError, NumericsError, FormatError, UsageError,
               CudaError, IgnisError)}


def raise_for(status: int, err: "abi.Error") -> None:
    if status == abi.IGN_OK:
        return
    msg = err.msg.decode(errors="replace")
    if status == abi.IGN_STEP_FAILURE:
        raise StepFailure(msg, err.stage, err.i, err.j, err.k)
    raise _BY_STATUS.get(status, IgnisError)(msg)
