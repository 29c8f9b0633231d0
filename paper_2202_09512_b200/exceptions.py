"""Error classes of the drop-in API.

Names and inheritance follow the reference hierarchy
(pkg/src/rescalkit/errors.py:4-21) so callers' exception handlers keep
working; the C-ABI status codes map onto them in ``_lib.check``.
"""


class RescalkitError(Exception):
    """Root of every error raised by this package."""


class DataError(RescalkitError):
    """Bad input: shapes, ranks, negative entries, zero norm (RK_ERR_DATA)."""


class NumericalError(RescalkitError):
    """A factor or the error trace became NaN/Inf (RK_ERR_NUMERICAL)."""


class GridError(RescalkitError):
    """Process-grid / NCCL misuse (RK_ERR_GRID)."""


class GridDeadlockError(GridError):
    """Ranks disagreed on the next collective (kept for API parity)."""
