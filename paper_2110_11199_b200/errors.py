"""Exception taxonomy of the reference (proj/include/adpsgd/errors.hpp:9-46), mapped 1:1
from the C ABI's adpsgd_status codes (include/adpsgd_b200.h)."""


class AdpsgdError(RuntimeError):
    code = -1


class InvalidOrderError(AdpsgdError, ValueError):
    code = 1


class DimensionError(AdpsgdError, ValueError):
    code = 2


class OutOfRegimeError(AdpsgdError):
    code = 3


class NumericalError(AdpsgdError):
    code = 4


class SyncViolationError(AdpsgdError):
    code = 5


class StalenessOverflowError(AdpsgdError):
    code = 6


class InvalidStateError(AdpsgdError):
    code = 7


class ConfigError(AdpsgdError):
    code = 8


class CudaError(AdpsgdError):
    code = 9


class NcclError(AdpsgdError):
    code = 10


BY_CODE = {c.code: c for c in (InvalidOrderError, DimensionError, OutOfRegimeError, NumericalError,
                               SyncViolationError, StalenessOverflowError, InvalidStateError, ConfigError,
                               CudaError, NcclError)}


def raise_for(code: int, message: str) -> None:
    if code == 0:
        return
    raise BY_CODE.get(code, AdpsgdError)(message or f"adpsgd status {code}")
