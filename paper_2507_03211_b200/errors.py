"""Exceptions of the drop-in (the class names and the tree are zosim's,
src/zosim/errors.py:8-56, so ``except`` clauses written for the reference
keep working).

Status codes returned by the C ABI (ZO_ERR_*, include/zo_b200.h) become
these classes in ``raise_for``; ``exit_code`` is the process status the
reference's CLI uses for each family (src/zosim/cli.py:176-192).

    ZosimError                     exit 1
    +-- ConfigurationError         exit 2   ABI status 2
    |   +-- DimensionError
    |   +-- MemoryCapacityError    (.block_id)
    +-- NumericError               exit 3   ABI status 3
    +-- FabricFault                exit 4
    |   +-- ConsistencyError
    +-- ProtocolError              exit 1   ABI status 1
    +-- SimulationError            exit 1
    +-- CudaError                  exit 1   ABI status 5 (native runtime failure; no reference analogue)
"""


class ZosimError(Exception): exit_code = 1                      # noqa: E701
class ConfigurationError(ZosimError): exit_code = 2             # noqa: E701
class DimensionError(ConfigurationError): pass                  # noqa: E701
class NumericError(ZosimError): exit_code = 3                   # noqa: E701
class FabricFault(ZosimError): exit_code = 4                    # noqa: E701
class ConsistencyError(FabricFault): pass                       # noqa: E701
class ProtocolError(ZosimError): pass                           # noqa: E701
class SimulationError(ZosimError): pass                         # noqa: E701
class CudaError(ZosimError): pass                               # noqa: E701


class MemoryCapacityError(ConfigurationError):
    def __init__(self, message, block_id=None):
        super().__init__(message)
        self.block_id = block_id


_BY_STATUS = {1: ProtocolError, 2: ConfigurationError, 3: NumericError, 4: FabricFault, 5: CudaError}


def raise_for(code: int, message: str) -> None:
    """Raise the class mapped to a nonzero ABI status (no-op for 0)."""
    if code:
        raise _BY_STATUS.get(code, ZosimError)(message)
