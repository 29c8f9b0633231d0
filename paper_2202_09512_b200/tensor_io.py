"""Tensor and factor files (drop-in for rescalkit.tensor's I/O, tensor.py:188-327).

Formats and bytes are the reference's: RSK1 dense binary, RSKM factor
matrices, and the ``%rescalk-coo`` text format. Loading a COO file runs the
native multithreaded parser of librescal_b200 (csrc/ingest.cpp; the
reference's loader is a pure-Python line loop, tensor.py:260-300), which
returns canonical per-slice CSR arrays with the reference's acceptance rules
and error texts. The binary formats are plain numpy reads/writes, as in the
reference.
"""

from __future__ import annotations

import ctypes
import os
import struct

import numpy as np
import scipy.sparse as sp

from . import _lib
from .containers import RelTensor, SparseRelTensor
from .exceptions import DataError

_DENSE_MAGIC = b"RSK1"
_MATRIX_MAGIC = b"RSKM"
_SPARSE_HEADER = "%rescalk-coo"
_FORMAT_VERSION = 1
_DTYPE_CODES = {0: np.float32, 1: np.float64}
_DTYPE_TO_CODE = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}
_HDR = "<IBQQ"


def save_tensor(t, path, format=None) -> None:
    """Write a tensor (tensor.py:188-201). Format defaults to the tensor's own
    representation."""
    if format is None:
        format = "sparse-coo" if isinstance(t, SparseRelTensor) else "dense-binary"
    if format == "dense-binary":
        if isinstance(t, SparseRelTensor):
            t = t.to_dense()
        _save_dense(t, path)
    elif format == "sparse-coo":
        if isinstance(t, RelTensor):
            raise DataError("convert to SparseRelTensor before sparse-coo save")
        _save_sparse(t, path)
    else:
        raise DataError(f"unknown format {format!r}")


def load_tensor(path, format=None):
    """Read a tensor (tensor.py:204-214); the format is inferred from the file
    when not given."""
    if format is None:
        with open(path, "rb") as f:
            head = f.read(4)
        format = "dense-binary" if head == _DENSE_MAGIC else "sparse-coo"
    if format == "dense-binary":
        return _load_dense(path)
    if format == "sparse-coo":
        return load_coo(path)
    raise DataError(f"unknown format {format!r}")


def _save_dense(t: RelTensor, path) -> None:
    code = _DTYPE_TO_CODE[t.slices.dtype]
    with open(path, "wb") as f:
        f.write(_DENSE_MAGIC)
        f.write(struct.pack(_HDR, _FORMAT_VERSION, code, t.n, t.m))
        f.write(np.ascontiguousarray(t.slices).tobytes())


def _load_dense(path) -> RelTensor:
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != _DENSE_MAGIC:
            raise DataError(f"malformed header: bad magic {magic!r}")
        header = f.read(struct.calcsize(_HDR))
        if len(header) != struct.calcsize(_HDR):
            raise DataError("malformed header: truncated")
        version, code, n, m = struct.unpack(_HDR, header)
        if version != _FORMAT_VERSION:
            raise DataError(f"unsupported format version {version}")
        if code not in _DTYPE_CODES:
            raise DataError(f"malformed header: unknown dtype code {code}")
        dtype = np.dtype(_DTYPE_CODES[code])
        expected = m * n * n * dtype.itemsize
        got = os.fstat(f.fileno()).st_size - f.tell()
        if got != expected:
            raise DataError(f"dimension mismatch: expected {expected} payload bytes, got {got}")
        arr = np.fromfile(f, dtype=dtype, count=m * n * n)
    return RelTensor(arr.reshape(m, n, n))


def _save_sparse(t: SparseRelTensor, path) -> None:
    lines = [f"{_SPARSE_HEADER} {t.n} {t.m} {t.nnz}\n"]
    for ti, s in enumerate(t.slices):
        coo = s.tocoo()
        order = np.lexsort((coo.col, coo.row))
        for r, c, v in zip(coo.row[order], coo.col[order], coo.data[order]):
            lines.append(f"{ti} {r} {c} {float(v)!r}\n")
    with open(path, "w", encoding="utf-8") as f:
        f.writelines(lines)


def load_coo(path) -> SparseRelTensor:
    """``%rescalk-coo`` text -> SparseRelTensor through the native parser."""
    lib = _lib.load()
    h = ctypes.c_void_p()
    n, m, nnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    rc = lib.rk_coo_open(str(path).encode(), ctypes.byref(h), ctypes.byref(n), ctypes.byref(m), ctypes.byref(nnz))
    if rc != 0:
        raise DataError(lib.rk_coo_last_error().decode())
    try:
        slices = []
        for t in range(m.value):
            cnt = lib.rk_coo_slice_nnz(h, t)
            indptr = np.empty(n.value + 1, dtype=np.int64)
            indices = np.empty(cnt, dtype=np.int32)
            data = np.empty(cnt, dtype=np.float64)
            rc = lib.rk_coo_fill(h, t, indptr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                 indices.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                 data.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
            if rc != 0:
                raise DataError("coo fill failed")
            idx_t = np.int32 if n.value < 2**31 else np.int64
            slices.append(sp.csr_matrix((data, indices.astype(idx_t, copy=False),
                                         indptr.astype(idx_t) if nnz.value < 2**31 else indptr),
                                        shape=(n.value, n.value)))
    finally:
        lib.rk_coo_close(h)
    return SparseRelTensor(slices, n=n.value)


def save_matrix(a, path) -> None:
    """Write a 2D factor matrix in the RSKM layout (tensor.py:303-313)."""
    a = np.asarray(a)
    if a.ndim != 2:
        raise DataError(f"expected a 2D matrix, got shape {a.shape}")
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    with open(path, "wb") as f:
        f.write(_MATRIX_MAGIC)
        f.write(struct.pack(_HDR, _FORMAT_VERSION, _DTYPE_TO_CODE[a.dtype], *a.shape))
        f.write(np.ascontiguousarray(a).tobytes())


def load_matrix(path) -> np.ndarray:
    """Read an RSKM factor matrix (tensor.py:316-327)."""
    with open(path, "rb") as f:
        if f.read(4) != _MATRIX_MAGIC:
            raise DataError("malformed header: bad magic")
        version, code, rows, cols = struct.unpack(_HDR, f.read(struct.calcsize(_HDR)))
        if version != _FORMAT_VERSION or code not in _DTYPE_CODES:
            raise DataError("malformed header")
        dtype = np.dtype(_DTYPE_CODES[code])
        payload = f.read()
    if len(payload) != rows * cols * dtype.itemsize:
        raise DataError("dimension mismatch in matrix payload")
    return np.frombuffer(payload, dtype=dtype).reshape(rows, cols).copy()
