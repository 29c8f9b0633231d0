"""Host-side tensor containers accepted by the drop-in API.

``RelTensor`` / ``SparseRelTensor`` keep the reference contracts
(pkg/src/rescalkit/tensor.py:45-139) so callers can switch without code
changes: a dense tensor is an (m, n, n) float32/float64 array with
non-negative entries, a sparse one is a list of canonical CSR slices
(duplicates summed, column indices sorted, explicit zeros dropped:
tensor.py:96-104, reproduced with the same scipy operations in the same
order so the index arrays are bit-identical). Error texts are the
reference's (tests compare them). The solver also takes the reference's own
objects (duck-typed on ``slices`` / ``m`` / ``n``). On the device a tensor
always lives as bf16 hi/lo planes.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .exceptions import DataError

# the reference's messages (tensor.py), shared by both containers
_MSG_NEGATIVE = "negative value in tensor"
_MSG_EMPTY = "sparse tensor needs at least one slice"
_MSG_SHAPES = "all slices must be square with identical shape"

# the CSR canonicalisation steps of tensor.py:96-104, in order
_CANONICAL_STEPS = ("sum_duplicates", "sort_indices", "eliminate_zeros")


class _SliceTensor:
    """Shared read-only view: m frontal n x n slices in ``self.slices``."""

    @property
    def dtype(self):
        first = self.slices[0] if isinstance(self.slices, list) else self.slices
        return first.dtype

    def slice_ops(self):
        return [self.slices[t] for t in range(self.m)]

    def _extra_repr(self) -> str:
        return ""

    def __repr__(self):
        return f"{type(self).__name__}(n={self.n}, m={self.m}{self._extra_repr()}, dtype={self.dtype})"


class RelTensor(_SliceTensor):
    """Dense relational tensor: m frontal n x n slices, all entries >= 0."""

    def __init__(self, slices):
        data = np.asarray(slices)
        if data.ndim != 3 or data.shape[1] != data.shape[2]:
            raise DataError(f"expected shape (m, n, n), got {data.shape}")
        if data.dtype != np.float32 and data.dtype != np.float64:
            data = data.astype(np.float64)
        if data.size > 0 and data.min() < 0:
            raise DataError(_MSG_NEGATIVE)
        self.slices = data
        self.m, self.n = int(data.shape[0]), int(data.shape[1])

    density = property(lambda self: 1.0)

    def astype(self, dtype) -> "RelTensor":
        return RelTensor(self.slices.astype(dtype))


def canonicalize_csr(s):
    """CSR index construction of tensor.py:96-104 (bit-exact: same scipy calls)."""
    csr = sp.csr_matrix(s)
    for step in _CANONICAL_STEPS:
        getattr(csr, step)()
    if csr.nnz > 0 and csr.data.min() < 0:
        raise DataError(_MSG_NEGATIVE)
    return csr


class SparseRelTensor(_SliceTensor):
    """Relational tensor with canonical CSR frontal slices."""

    def __init__(self, slices, n=None):
        if not slices:
            raise DataError(_MSG_EMPTY)
        canonical = list(map(canonicalize_csr, slices))
        rows, cols = canonical[0].shape
        if rows != cols or any(c.shape != (rows, cols) for c in canonical):
            raise DataError(_MSG_SHAPES)
        if n is not None and n != rows:
            raise DataError(f"dimension mismatch: header n={n}, slices are {rows}")
        self.slices = canonical
        self.n, self.m = rows, len(canonical)

    @property
    def nnz(self) -> int:
        return int(sum(c.nnz for c in self.slices))

    @property
    def density(self) -> float:
        return self.nnz / (self.n * self.n * self.m)

    def _extra_repr(self) -> str:
        return f", nnz={self.nnz}"

    def to_dense(self) -> RelTensor:
        return RelTensor(np.stack([np.asarray(c.todense()) for c in self.slices]))


def fro_norm(t) -> float:
    """sqrt of the fp64 sum of squares (tensor.py:173-181)."""
    if is_sparse(t):
        total = 0.0
        for c in t.slices:
            total += float(np.sum(c.data.astype(np.float64) ** 2))
        return float(np.sqrt(total))
    return float(np.sqrt(np.sum(np.asarray(t.slices, dtype=np.float64) ** 2)))


def is_sparse(x) -> bool:
    parts = getattr(x, "slices", None)
    return isinstance(parts, (list, tuple)) and len(parts) > 0 and sp.issparse(parts[0])


def dense_slices(x) -> np.ndarray:
    """(m, n, n) host array of any accepted tensor (sparse densified)."""
    if is_sparse(x):
        return np.stack([np.asarray(c.toarray()) for c in x.slices])
    data = np.asarray(x.slices)
    if data.ndim != 3:
        raise DataError(f"expected (m, n, n) slices, got {data.shape}")
    return data


def tensor_dtype(x):
    return np.dtype(x.dtype)
