"""Error hierarchy of the reference (include/rectri/error.hpp:10-84), one class
per reference exception type, plus CudaError for device failures (no
reference twin).  Status codes come from include/rectri_cu.h."""
from __future__ import annotations


class Error(RuntimeError):
    """Root of the library's failure hierarchy (error.hpp:11-14)."""


class ShapeError(Error):
    """Non-conforming matrix dimensions (error.hpp:17-20)."""


class BoundsError(Error):
    """Requested subview rectangle escapes its parent (error.hpp:23-26)."""


class AliasError(Error):
    """Output view overlaps a read-only input view (error.hpp:29-32)."""


class SplitError(Error):
    """split_half called with n < 2 (error.hpp:35-38)."""


class TileLimitError(Error):
    """Base kernel invoked on a tile larger than its limit (error.hpp:41-44)."""


class ConfigError(Error):
    """Invalid flags, threshold, backend or bench configuration (error.hpp:47-50)."""


class SingularityError(Error):
    """Exactly-zero pivot in a NonUnit solve; ``index`` is the row of the zero
    diagonal entry, global for the recursive drivers (error.hpp:55-66)."""

    def __init__(self, index: int, message: str | None = None):
        super().__init__(message or f"singular triangular matrix: zero diagonal at row {index}")
        self._index = int(index)

    def index(self) -> int:
        return self._index


class ValidationError(Error):
    """Benchmark result failed its residual gate (error.hpp:69-72)."""


class JoinError(Error):
    """Ratio report inputs do not share the same key set (error.hpp:75-78)."""


class IoError(Error):
    """Unreadable or unwritable file path (error.hpp:81-84)."""


class CudaError(Error):
    """CUDA runtime or launch failure inside the device library."""


STATUS_OK = 0
_BY_STATUS = {
    1: ConfigError,
    2: ShapeError,
    3: AliasError,
    5: TileLimitError,
    6: CudaError,
    7: BoundsError,
    8: SplitError,
}


def raise_for_status(status: int, message: str, singular_row: int = -1) -> None:
    if status == STATUS_OK:
        return
    if status == 4:
        raise SingularityError(singular_row, message or None)
    cls = _BY_STATUS.get(status, Error)
    raise cls(message)
