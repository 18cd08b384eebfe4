"""The reference error taxonomy (proj/core/include/pbrl/errors.hpp:9-48) mapped from C-ABI codes."""


class PbrlError(Exception):
    """Base class of every error raised by the population API."""


class ShapeError(PbrlError, ValueError):
    """Tensor extents do not line up (errors.hpp:9)."""


class ConfigError(PbrlError, ValueError):
    """A configuration value is out of its legal range (errors.hpp:15)."""


class UsageError(PbrlError, RuntimeError):
    """API misuse: bad index, stale state (errors.hpp:21)."""


class NotReadyError(PbrlError, RuntimeError):
    """The requested value does not exist yet (errors.hpp:27)."""


class ResourceError(PbrlError, MemoryError):
    """Estimated or actual memory footprint exceeds what is available (errors.hpp:33)."""


class DataStarvationError(PbrlError, RuntimeError):
    """A sampler ran dry inside update_k_steps (errors.hpp:39, algos.hpp:958-962)."""


class DegeneratePopulationError(PbrlError, RuntimeError):
    """DvD kernel matrix not positive definite even with jitter (errors.hpp:45)."""


class CudaError(PbrlError, RuntimeError):
    """A CUDA runtime call failed."""


class NcclError(PbrlError, RuntimeError):
    """A collective failed."""


_CODES = {-1: ShapeError, -2: ConfigError, -3: UsageError, -4: NotReadyError, -5: ResourceError,
          -6: DataStarvationError, -7: CudaError, -8: NcclError, -9: DegeneratePopulationError}


def raise_for(code: int, message: str) -> None:
    raise _CODES.get(code, PbrlError)(message)
