"""Exception classes mirroring slap::Error and its kinds (reference
proj/core/include/slap/error.hpp:10-36).  The C-ABI returns status codes; the
host layer raises the matching class, whose ``kind`` is the reference's stable
error name."""
from __future__ import annotations


class Error(RuntimeError):
    kind = "Error"

    def __init__(self, msg: str = ""):
        super().__init__(f"{self.kind}: {msg}")


class NameError_(Error):
    kind = "NameError"


class DimError(Error):
    kind = "DimError"


class IndexError_(Error):
    kind = "IndexError"


class ShapeError(Error):
    kind = "ShapeError"


class ArityError(Error):
    kind = "ArityError"


class DeadlockError(Error):
    kind = "DeadlockError"


class BudgetError(Error):
    kind = "BudgetError"


class InternalError(Error):
    kind = "InternalError"


class CudaError(Error):
    kind = "CudaError"


class InvalidArgument(Error):
    kind = "InvalidArgument"


class OutOfMemory(Error):
    kind = "OutOfMemory"


class StochasticityError(Error):
    kind = "StochasticityError"


class IoError(Error):
    kind = "IoError"


class FormatError(Error):
    kind = "FormatError"


BY_STATUS = {
    1: DimError,
    2: ShapeError,
    3: InternalError,
    4: NameError_,
    5: BudgetError,
    6: IndexError_,
    7: InvalidArgument,
    8: CudaError,
    9: OutOfMemory,
    10: DeadlockError,
    11: StochasticityError,
    12: IoError,
    13: FormatError,
}
