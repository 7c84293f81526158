"""Exception taxonomy of the reference (proj/include/hsdla/errors.hpp:9-26), mapped
from the C-ABI status codes."""
from . import _lib


class DimensionError(ValueError):
    """Operand shapes do not conform (errors.hpp:9-12)."""


class SizingError(RuntimeError):
    """Allocation would overflow / does not fit (errors.hpp:14-17)."""


class ConfigError(RuntimeError):
    """Invalid device / strategy configuration (errors.hpp:19-22)."""


class IoError(RuntimeError):
    """File format or filesystem failure (errors.hpp:24-27)."""


class CudaError(RuntimeError):
    """CUDA runtime / kernel launch failure."""


class NcclError(RuntimeError):
    """NCCL failure."""


_BY_CODE = {
    _lib.DIMENSION_ERROR: DimensionError,
    _lib.SIZING_ERROR: SizingError,
    _lib.CONFIG_ERROR: ConfigError,
    _lib.IO_ERROR: IoError,
    _lib.CUDA_ERROR: CudaError,
    _lib.NCCL_ERROR: NcclError,
}


def check(rc, what=""):
    if rc != _lib.OK:
        raise _BY_CODE.get(rc, RuntimeError)(f"{what}: {_lib.last_error()}" if what else _lib.last_error())
