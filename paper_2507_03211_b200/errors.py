"""Exception hierarchy of the drop-in, mirroring src/zosim/errors.py:8-56.

The C ABI returns ZO_ERR_* status codes (include/zo_b200.h); ``raise_for``
maps them onto these classes so callers catch exactly what they caught with
the reference.  Exit codes follow src/zosim/cli.py:176-192.
"""


class ZosimError(Exception):
    """Base class (errors.py:8)."""


class ConfigurationError(ZosimError):
    exit_code = 2


class DimensionError(ConfigurationError):
    """Shape mismatch (errors.py:18-20)."""


class MemoryCapacityError(ConfigurationError):
    def __init__(self, message, block_id=None):
        super().__init__(message)
        self.block_id = block_id


class NumericError(ZosimError):
    exit_code = 3


class FabricFault(ZosimError):
    exit_code = 4


class ConsistencyError(FabricFault):
    """Replicas diverged (errors.py:43-44)."""


class ProtocolError(ZosimError):
    exit_code = 1


class SimulationError(ZosimError):
    exit_code = 1


class CudaError(ZosimError):
    """CUDA runtime failure inside the native library (no reference analogue)."""

    exit_code = 1


_BY_CODE = {1: ProtocolError, 2: ConfigurationError, 3: NumericError, 4: FabricFault, 5: CudaError}


def raise_for(code: int, message: str) -> None:
    if code:
        raise _BY_CODE.get(code, ZosimError)(message)
