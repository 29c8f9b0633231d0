"""Tensor and factor files in the reference's formats (tensor.py:188-327).

Formats (byte-compatible with rescalkit):
  * RSK1 dense tensor: magic ``RSK1``, little-endian record (u32 version,
    u8 dtype code, u64 n, u64 m), then the (m, n, n) C-ordered payload;
  * RSKM factor matrix: magic ``RSKM``, the same record with (rows, cols);
  * ``%rescalk-coo n m nnz`` text, one ``t i j value`` line per stored entry.

Implementation: the RSK1 payload is memory-mapped (``DenseFile``), so a grid
rank can read only its own block (``multigpu.BlockSource.from_file``) and a
whole-tensor load is one sequential read. COO files are parsed by the native
multithreaded parser of librescal_b200 (csrc/ingest.cpp) straight into
canonical per-slice CSR arrays with the reference's acceptance rules and error
texts (the reference loops over lines in Python, tensor.py:260-300). Error
messages match the reference's so callers' exception handling carries over.
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

_VERSION = 1
_CODE_TO_DTYPE = {0: np.dtype(np.float32), 1: np.dtype(np.float64)}
_DTYPE_TO_CODE = {v: k for k, v in _CODE_TO_DTYPE.items()}
_RECORD = struct.Struct("<IBQQ")  # version, dtype code, dim0, dim1 (after the 4-byte magic)
_COO_TAG = "%rescalk-coo"


def _write_record(f, magic: bytes, dtype, d0: int, d1: int) -> None:
    f.write(magic + _RECORD.pack(_VERSION, _DTYPE_TO_CODE[np.dtype(dtype)], int(d0), int(d1)))


class DenseFile:
    """A dense RSK1 file opened for reading: header checked, payload mapped
    read-only as ``array`` (m, n, n) without reading it."""

    def __init__(self, path):
        size = os.path.getsize(path)
        with open(path, "rb") as f:
            magic = f.read(4)
            if magic != b"RSK1":
                raise DataError(f"malformed header: bad magic {magic!r}")
            raw = f.read(_RECORD.size)
        if len(raw) != _RECORD.size:
            raise DataError("malformed header: truncated")
        version, code, n, m = _RECORD.unpack(raw)
        if version != _VERSION:
            raise DataError(f"unsupported format version {version}")
        if code not in _CODE_TO_DTYPE:
            raise DataError(f"malformed header: unknown dtype code {code}")
        self.n, self.m, self.dtype = int(n), int(m), _CODE_TO_DTYPE[code]
        offset = 4 + _RECORD.size
        expected = self.m * self.n * self.n * self.dtype.itemsize
        if size - offset != expected:
            raise DataError(f"dimension mismatch: expected {expected} payload bytes, got {size - offset}")
        self.array = (np.memmap(path, dtype=self.dtype, mode="r", offset=offset, shape=(self.m, self.n, self.n))
                      if expected else np.zeros((self.m, self.n, self.n), dtype=self.dtype))

    def tensor(self) -> RelTensor:
        return RelTensor(np.array(self.array))


def _coo_lines(t: SparseRelTensor):
    yield f"{_COO_TAG} {t.n} {t.m} {t.nnz}\n"
    for ti, s in enumerate(t.slices):
        c = s.tocoo()
        order = np.lexsort((c.col, c.row))  # row-major entry order
        rows, cols, vals = c.row[order], c.col[order], c.data[order]
        for lo in range(0, len(order), 1 << 16):
            hi = lo + (1 << 16)
            yield "".join(f"{ti} {r} {j} {float(v)!r}\n"
                          for r, j, v in zip(rows[lo:hi].tolist(), cols[lo:hi].tolist(), vals[lo:hi].tolist()))


def _write_dense(t, path) -> None:
    if isinstance(t, SparseRelTensor):
        t = t.to_dense()
    arr = np.ascontiguousarray(t.slices)
    with open(path, "wb") as f:
        _write_record(f, b"RSK1", arr.dtype, t.n, t.m)
        arr.tofile(f)


def _write_coo(t, path) -> None:
    if isinstance(t, RelTensor):
        raise DataError("convert to SparseRelTensor before sparse-coo save")
    with open(path, "w", encoding="utf-8") as f:
        f.writelines(_coo_lines(t))


_WRITERS = {"dense-binary": _write_dense, "sparse-coo": _write_coo}


def save_tensor(t, path, format=None) -> None:
    """Write a tensor (tensor.py:188-201); the format defaults to the tensor's
    own representation."""
    fmt = format or ("sparse-coo" if isinstance(t, SparseRelTensor) else "dense-binary")
    if fmt not in _WRITERS:
        raise DataError(f"unknown format {format!r}")
    _WRITERS[fmt](t, path)


def load_tensor(path, format=None):
    """Read a tensor (tensor.py:204-214); the format is sniffed from the first
    four bytes when not given."""
    if format is None:
        with open(path, "rb") as f:
            format = "dense-binary" if f.read(4) == b"RSK1" else "sparse-coo"
    if format == "dense-binary":
        return DenseFile(path).tensor()
    if format == "sparse-coo":
        return load_coo(path)
    raise DataError(f"unknown format {format!r}")


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
    """Write a 2D factor matrix as RSKM (tensor.py:303-313)."""
    a = np.asarray(a)
    if a.ndim != 2:
        raise DataError(f"expected a 2D matrix, got shape {a.shape}")
    if a.dtype not in _DTYPE_TO_CODE:
        a = a.astype(np.float64)
    with open(path, "wb") as f:
        _write_record(f, b"RSKM", a.dtype, *a.shape)
        np.ascontiguousarray(a).tofile(f)


def load_matrix(path) -> np.ndarray:
    """Read an RSKM factor matrix (tensor.py:316-327)."""
    raw = np.fromfile(path, dtype=np.uint8)
    if raw[:4].tobytes() != b"RSKM":
        raise DataError("malformed header: bad magic")
    head = raw[4:4 + _RECORD.size].tobytes()
    if len(head) != _RECORD.size:
        raise DataError("malformed header")
    version, code, rows, cols = _RECORD.unpack(head)
    if version != _VERSION or code not in _CODE_TO_DTYPE:
        raise DataError("malformed header")
    dtype = _CODE_TO_DTYPE[code]
    payload = raw[4 + _RECORD.size:]
    if payload.size != rows * cols * dtype.itemsize:
        raise DataError("dimension mismatch in matrix payload")
    return payload.view(dtype).reshape(rows, cols).copy()
