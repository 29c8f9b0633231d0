"""Host-side tensor containers accepted by the drop-in API.

``RelTensor`` / ``SparseRelTensor`` follow the reference contracts
(pkg/src/rescalkit/tensor.py:45-139): dense (m, n, n) float32/float64 with
non-negative entries; sparse = one canonical CSR per slice (duplicates summed,
column indices sorted, explicit zeros dropped — tensor.py:96-104). The solver
also accepts the reference's own objects (duck-typed on ``slices``/``m``/``n``).
On the device the tensor always lives as bf16 hi/lo planes.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .exceptions import DataError


class RelTensor:
    """Dense relational tensor: m frontal n x n slices, all entries >= 0."""

    def __init__(self, slices):
        arr = np.asarray(slices)
        if arr.ndim != 3 or arr.shape[1] != arr.shape[2]:
            raise DataError(f"expected shape (m, n, n), got {arr.shape}")
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        if arr.size and arr.min() < 0:
            raise DataError("negative value in tensor")
        self.slices = arr
        self.m, self.n = arr.shape[0], arr.shape[1]

    @property
    def dtype(self):
        return self.slices.dtype

    @property
    def density(self) -> float:
        return 1.0

    def slice_ops(self):
        return [self.slices[t] for t in range(self.m)]

    def astype(self, dtype) -> "RelTensor":
        return RelTensor(self.slices.astype(dtype))

    def __repr__(self):
        return f"RelTensor(n={self.n}, m={self.m}, dtype={self.dtype})"


def canonicalize_csr(s):
    """CSR index construction of tensor.py:96-104 (bit-exact: same scipy calls)."""
    c = sp.csr_matrix(s)
    c.sum_duplicates()
    c.sort_indices()
    c.eliminate_zeros()
    if c.nnz and c.data.min() < 0:
        raise DataError("negative value in tensor")
    return c


class SparseRelTensor:
    """Relational tensor with canonical CSR frontal slices."""

    def __init__(self, slices, n=None):
        if not slices:
            raise DataError("sparse tensor needs at least one slice")
        canon = [canonicalize_csr(s) for s in slices]
        shape = canon[0].shape
        if shape[0] != shape[1] or any(c.shape != shape for c in canon):
            raise DataError("all slices must be square with identical shape")
        if n is not None and n != shape[0]:
            raise DataError(f"dimension mismatch: header n={n}, slices are {shape[0]}")
        self.slices = canon
        self.n = shape[0]
        self.m = len(canon)

    @property
    def dtype(self):
        return self.slices[0].dtype

    @property
    def nnz(self) -> int:
        return sum(s.nnz for s in self.slices)

    @property
    def density(self) -> float:
        return self.nnz / (self.n * self.n * self.m)

    def slice_ops(self):
        return list(self.slices)

    def to_dense(self) -> RelTensor:
        return RelTensor(np.stack([np.asarray(s.todense()) for s in self.slices]))

    def __repr__(self):
        return f"SparseRelTensor(n={self.n}, m={self.m}, nnz={self.nnz}, dtype={self.dtype})"


def fro_norm(t) -> float:
    """sqrt of the fp64 sum of squares (tensor.py:173-181)."""
    if is_sparse(t):
        return float(np.sqrt(sum(float(np.sum(s.data.astype(np.float64) ** 2)) for s in t.slices)))
    return float(np.sqrt(np.sum(np.asarray(t.slices, dtype=np.float64) ** 2)))


def is_sparse(x) -> bool:
    s = getattr(x, "slices", None)
    return isinstance(s, (list, tuple)) and len(s) > 0 and sp.issparse(s[0])


def dense_slices(x) -> np.ndarray:
    """(m, n, n) host array of any accepted tensor (sparse densified)."""
    if is_sparse(x):
        return np.stack([np.asarray(s.toarray()) for s in x.slices])
    arr = np.asarray(x.slices)
    if arr.ndim != 3:
        raise DataError(f"expected (m, n, n) slices, got {arr.shape}")
    return arr


def tensor_dtype(x):
    return np.dtype(x.dtype)
