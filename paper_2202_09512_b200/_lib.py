"""ctypes binding of librescal_b200.so (include/rescal_b200.h).

The product path has no CPU fallback: if the CUDA library is missing or no
Blackwell GPU is visible, every solver entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .exceptions import DataError, GridError, NumericalError, RescalkitError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librescal_b200.so")

RK_OK, RK_ERR_DATA, RK_ERR_NUMERICAL, RK_ERR_GRID, RK_ERR_DEVICE = range(5)
RK_F32, RK_F64 = 0, 1
ENGINES = {"auto": 0, "tc": 1, "simt": 2}


class DeviceError(RescalkitError):
    """CUDA / NCCL failure inside the engine (no reference equivalent)."""


_EXC = {RK_ERR_DATA: DataError, RK_ERR_NUMERICAL: NumericalError, RK_ERR_GRID: GridError,
        RK_ERR_DEVICE: DeviceError}

_i32, _i64, _u64, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
_vp = ctypes.c_void_p
_pd = ctypes.POINTER(ctypes.c_double)
_pi32 = ctypes.POINTER(ctypes.c_int32)
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pf = ctypes.POINTER(ctypes.c_float)

# name -> (restype, argtypes); mirrors include/rescal_b200.h plus the
# engine-private helpers declared at the end of this table.
SIGNATURES = {
    "rk_version": (ctypes.c_int, []),
    "rk_last_error": (ctypes.c_char_p, []),
    "rk_device_count": (ctypes.c_int, [_pi32]),
    "rk_create": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i32, _i32, ctypes.POINTER(_vp)]),
    "rk_destroy": (None, [_vp]),
    "rk_upload_dense": (ctypes.c_int, [_vp, _vp, _i32]),
    "rk_upload_block": (ctypes.c_int, [_vp, _vp, _i32, _i64, _i64, _f64]),
    "rk_create_sparse": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i32, ctypes.POINTER(_vp)]),
    "rk_upload_csr": (ctypes.c_int, [_vp, _pi64, ctypes.POINTER(ctypes.c_int32), _vp, _i32, _i64]),
    "rk_upload_csr_slices": (ctypes.c_int, [_vp, _vp, _vp, _vp, _pi64, _i32]),
    "rk_fill_uniform": (ctypes.c_int, [_vp, _u64]),
    "rk_set_factors": (ctypes.c_int, [_vp, _pd, _pd]),
    "rk_get_factors": (ctypes.c_int, [_vp, _pd, _pd]),
    "rk_run": (ctypes.c_int, [_vp, _i32, _f64, _i32, _f64, _pd, _pi32]),
    "rk_update_r": (ctypes.c_int, [_vp, _f64]),
    "rk_update_a": (ctypes.c_int, [_vp, _f64]),
    "rk_residual": (ctypes.c_int, [_vp, _pd, _pd]),
    "rk_regress_r": (ctypes.c_int, [_vp, _i32, _f64, _f64, _pi32]),
    "rk_perturb": (ctypes.c_int, [_vp, _u64, _u64, _u64, _u64, _f64, _i64, _i64, _i64, _pi64]),
    "rk_grid_init": (ctypes.c_int, [_vp, _i32, _i32, _i32, _vp, _i64]),
    "rk_nccl_unique_id": (ctypes.c_int, [_vp]),
    "rk_tensor_export": (ctypes.c_int, [_vp, _vp, _i32]),
    "rk_tensor_import": (ctypes.c_int, [_vp, _vp]),
    "rk_last_timing": (ctypes.c_int, [_vp, _pd, _i32]),
    "rk_stream": (_vp, [_vp]),
    "rk_info": (ctypes.c_int, [_vp, _pi64, _i32]),
    # engine-private (not part of the reference-facing header)
    "rk_set_rank": (ctypes.c_int, [_vp, _i32]),
    "rk_set_option": (ctypes.c_int, [_vp, _i32, _i64]),
    "rk_uniform_values": (ctypes.c_int, [_u64, _i64, _i64, _pf]),
    "rk_pcg64_draws": (ctypes.c_int, [_u64, _u64, _u64, _u64, _u64, _i64, _pd]),
    "rk_pcg64_draws_on": (ctypes.c_int, [_i32, _u64, _u64, _u64, _u64, _u64, _i64, _pd]),
    "rk_coo_open": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(_i64),
                                   ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "rk_coo_last_error": (ctypes.c_char_p, []),
    "rk_coo_slice_nnz": (_i64, [_vp, _i64]),
    "rk_coo_fill": (ctypes.c_int, [_vp, _i64, _pi64, ctypes.POINTER(ctypes.c_int32), _pd]),
    "rk_coo_close": (None, [_vp]),
    "rk_release_cached_memory": (None, []),
    "rk_gram_apply": (ctypes.c_int, [_vp, _pd, _i32, _pd]),
    "rk_unfold_sign_norms": (ctypes.c_int, [_vp, _pd, _i32, _pd, _pd]),
    "rk_positive_mean": (ctypes.c_int, [_vp, _pd]),
    "rk_perturb_values": (ctypes.c_int, [_i32, _u64, _u64, _u64, _u64, _f64, _i32, _vp, _i64, _u64, _i32]),
    "rk_perturb_csr_values": (ctypes.c_int, [_i32, _u64, _u64, _u64, _u64, _f64, _i32, _i64, _i64, _pi64,
                                             ctypes.POINTER(ctypes.c_int32), _vp, _i64]),
    "rk_grid_block": (ctypes.c_int, [_vp, _pi64, _i32]),
    "rk_grid_colmap": (ctypes.c_int, [_vp, _pi64]),
    "rk_time_k1": (ctypes.c_int, [_vp, _i32, _pd]),
    "rk_trace_len": (ctypes.c_int, [_vp, _pi32]),
    "rk_restore": (ctypes.c_int, [_vp]),
    "rk_phase_timing": (ctypes.c_int, [_vp, _pd, _i32]),
    "rk_block_uniform": (ctypes.c_int, [_vp, _u64, _pf]),
    "rk_csc_copy": (ctypes.c_int, [_vp, _pi64, ctypes.POINTER(ctypes.c_int32), _pf]),
    "rk_csr_copy": (ctypes.c_int, [_vp, _pi64, ctypes.POINTER(ctypes.c_int32), _pf]),
    "rk_fill_sparse_uniform": (ctypes.c_int, [_vp, _u64, _i64]),
    "rk_nnz": (ctypes.c_int, [_vp, _pi64]),
    "rk_debug_guards": (ctypes.c_int, [_i32]),
    "rk_debug_check_guards": (ctypes.c_int, [_pi64, _pi64]),
    "rk_debug_overrun": (ctypes.c_int, [_i64]),
    "rk_debug_read_pq": (ctypes.c_int, [_vp, _vp, _vp]),
}

_LIB = None


def load():
    """Load the CUDA library (raises ImportError when it was never built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.environ.get("RK_LIB_PATH", LIB_PATH)  # experiments: an alternative in-tree build
    if not os.path.exists(path):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the RESCAL engine has no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        if path != LIB_PATH and not hasattr(lib, name):
            continue  # an older experimental build
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(status):
    if status != RK_OK:
        msg = load().rk_last_error().decode(errors="replace")
        raise _EXC.get(status, RescalkitError)(msg)


def _dp(a):
    return a.ctypes.data_as(_pd)


def pcg64_seed_state(entropy):
    """numpy PCG64 (state, inc) after seeding from SeedSequence(entropy), as
    four u64 words (state_hi, state_lo, inc_hi, inc_lo) — the published
    seeding of the reference's RNG (dist_rescal.py:167-168)."""
    bg = np.random.PCG64(np.random.SeedSequence(entropy))
    st = bg.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return (s >> 64) & m, s & m, (inc >> 64) & m, inc & m


class Engine:
    """One device-resident RESCAL problem (tensor + factors) on one GPU."""

    def __init__(self, n, m, k, device=None, engine="auto", sparse=False):
        lib = load()
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0"))
        self.n, self.m, self.k = int(n), int(m), int(k)
        self.sparse = bool(sparse)
        self.device = int(device)
        self._h = _vp()
        if self.sparse:
            check(lib.rk_create_sparse(int(device), self.n, self.m, self.k, ctypes.byref(self._h)))
        else:
            check(lib.rk_create(int(device), self.n, self.m, self.k, ENGINES[engine], ctypes.byref(self._h)))
        self._lib = lib

    # lifecycle -----------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.rk_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # data ------------------------------------------------------------------
    def upload(self, x):
        x = np.ascontiguousarray(x)
        if x.dtype not in (np.float32, np.float64):
            x = x.astype(np.float64)
        if x.shape != (self.m, self.n, self.n):
            raise DataError(f"tensor shape {x.shape} != ({self.m}, {self.n}, {self.n})")
        check(self._lib.rk_upload_dense(self._h, x.ctypes.data_as(_vp), RK_F32 if x.dtype == np.float32 else RK_F64))

    def upload_csr(self, slices):
        """Canonical CSR slices (scipy) -> device CSR + device-built CSC.

        The per-slice arrays are handed over as they are (no concatenation);
        the library streams them through a pinned ring and validates them on
        the device."""
        if len(slices) != self.m:
            raise DataError(f"expected {self.m} slices, got {len(slices)}")
        keep = []
        dts = {s.data.dtype for s in slices}
        dt = np.float32 if dts == {np.dtype(np.float32)} else np.float64
        ip = (ctypes.c_void_p * self.m)()
        ix = (ctypes.c_void_p * self.m)()
        dv = (ctypes.c_void_p * self.m)()
        nnz = np.empty(self.m, dtype=np.int64)
        for t, sl in enumerate(slices):
            a = np.ascontiguousarray(sl.indptr, dtype=np.int64)
            b = np.ascontiguousarray(sl.indices, dtype=np.int32)
            c = np.ascontiguousarray(sl.data, dtype=dt)
            keep += [a, b, c]
            ip[t], ix[t], dv[t] = a.ctypes.data, b.ctypes.data, c.ctypes.data
            nnz[t] = sl.nnz
        check(self._lib.rk_upload_csr_slices(self._h, ctypes.cast(ip, _vp), ctypes.cast(ix, _vp),
                                             ctypes.cast(dv, _vp), nnz.ctypes.data_as(_pi64),
                                             RK_F32 if dt == np.float32 else RK_F64))
        del keep

    # ---- NNDSVD support (products with the unfolding M = [X_t | X_t^T]) ----
    def gram_apply(self, v: np.ndarray) -> np.ndarray:
        """Y = M M^T V for an (n, b) block V (fp64 result)."""
        v = np.ascontiguousarray(v, dtype=np.float64)
        y = np.empty_like(v)
        check(self._lib.rk_gram_apply(self._h, _dp(v), int(v.shape[1]), _dp(y)))
        return y

    def unfold_sign_norms(self, u: np.ndarray):
        """Squared norms of the positive / negative parts of each column of M^T U."""
        u = np.ascontiguousarray(u, dtype=np.float64)
        pos = np.empty(u.shape[1])
        neg = np.empty(u.shape[1])
        check(self._lib.rk_unfold_sign_norms(self._h, _dp(u), int(u.shape[1]), _dp(pos), _dp(neg)))
        return pos, neg

    def positive_mean(self) -> float:
        out = _f64(0.0)
        check(self._lib.rk_positive_mean(self._h, ctypes.byref(out)))
        return float(out.value)

    def fill_sparse_uniform(self, seed, nnz_per_slice):
        """Synthetic uniform-random sparse slices generated on the device."""
        check(self._lib.rk_fill_sparse_uniform(self._h, int(seed), int(nnz_per_slice)))

    @property
    def nnz(self):
        out = _i64(0)
        check(self._lib.rk_nnz(self._h, ctypes.byref(out)))
        return int(out.value)

    def csr_arrays(self):
        nnz = self.nnz
        indptr = np.empty(self.m * (self.n + 1), dtype=np.int64)
        indices = np.empty(nnz, dtype=np.int32)
        data = np.empty(nnz, dtype=np.float32)
        check(self._lib.rk_csr_copy(self._h, indptr.ctypes.data_as(_pi64),
                                    indices.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                    data.ctypes.data_as(_pf)))
        return indptr.reshape(self.m, self.n + 1), indices, data

    def csc_arrays(self, nnz):
        """Device-built CSC (tests: index construction must match scipy)."""
        indptr = np.empty(self.m * (self.n + 1), dtype=np.int64)
        indices = np.empty(nnz, dtype=np.int32)
        data = np.empty(nnz, dtype=np.float32)
        check(self._lib.rk_csc_copy(self._h, indptr.ctypes.data_as(_pi64),
                                    indices.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                    data.ctypes.data_as(_pf)))
        return indptr.reshape(self.m, self.n + 1), indices, data

    def upload_block(self, xb, sq_norm_global):
        xb = np.ascontiguousarray(xb)
        if xb.dtype not in (np.float32, np.float64):
            xb = xb.astype(np.float64)
        check(self._lib.rk_upload_block(self._h, xb.ctypes.data_as(_vp),
                                        RK_F32 if xb.dtype == np.float32 else RK_F64,
                                        xb.shape[1], xb.shape[2], float(sq_norm_global)))

    def fill_uniform(self, seed):
        check(self._lib.rk_fill_uniform(self._h, int(seed)))

    def set_rank(self, k):
        check(self._lib.rk_set_rank(self._h, int(k)))
        self.k = int(k)

    def set_option(self, key, value):
        check(self._lib.rk_set_option(self._h, int(key), int(value)))

    def set_factors(self, a, r):
        a = np.ascontiguousarray(a, dtype=np.float64)
        r = np.ascontiguousarray(r, dtype=np.float64)
        if a.shape != (self.n, self.k) or r.shape != (self.m, self.k, self.k):
            raise DataError("initial factors do not match tensor/k")
        check(self._lib.rk_set_factors(self._h, _dp(a), _dp(r)))

    def get_factors(self):
        a = np.empty((self.n, self.k), dtype=np.float64)
        r = np.empty((self.m, self.k, self.k), dtype=np.float64)
        check(self._lib.rk_get_factors(self._h, _dp(a), _dp(r)))
        return a, r

    def debug_read_pq(self):
        """P = X_t A and Q = X_t^T A of the last K1 pass, [m][n_pad][k_pad] fp32."""
        inf = self.info()
        shape = (self.m, inf["n_pad"], inf["k_pad"])
        p = np.empty(shape, dtype=np.float32)
        q = np.empty(shape, dtype=np.float32)
        check(self._lib.rk_debug_read_pq(self._h, p.ctypes.data, q.ctypes.data))
        return p, q

    # compute ---------------------------------------------------------------
    def run(self, iters, eps, track_error=True, tol=None):
        trace = np.zeros(iters + 1, dtype=np.float64)
        done = _i32(0)
        status = self._lib.rk_run(self._h, int(iters), float(eps), 1 if track_error else 0,
                                  -1.0 if tol is None else float(tol), _dp(trace), ctypes.byref(done))
        tl = _i32(0)
        self._lib.rk_trace_len(self._h, ctypes.byref(tl))
        self.last_trace = trace[: tl.value].copy() if track_error else np.zeros(0)
        check(status)
        return int(done.value), self.last_trace

    def update_r(self, eps):
        check(self._lib.rk_update_r(self._h, float(eps)))

    def update_a(self, eps):
        check(self._lib.rk_update_a(self._h, float(eps)))

    def residual(self):
        res, nrm = _f64(0.0), _f64(0.0)
        check(self._lib.rk_residual(self._h, ctypes.byref(res), ctypes.byref(nrm)))
        return res.value, nrm.value

    def regress_r(self, max_iters, tol, eps):
        done = _i32(0)
        check(self._lib.rk_regress_r(self._h, int(max_iters), -1.0 if tol is None else float(tol),
                                     float(eps), ctypes.byref(done)))
        return int(done.value)

    def perturb(self, entropy, delta, n_global=None, row0=0):
        sh, sl, ih, il = pcg64_seed_state(entropy)
        check(self._lib.rk_perturb(self._h, sh, sl, ih, il, float(delta),
                                   int(n_global or self.n), int(row0), 0, None))

    def block_uniform(self, seed, rows, cols):
        """Exact fp32 values of this engine's block of the synthetic tensor."""
        out = np.empty((self.m, rows, cols), dtype=np.float32)
        check(self._lib.rk_block_uniform(self._h, int(seed), out.ctypes.data_as(_pf)))
        return out

    def restore(self):
        """Undo rk_perturb: the device tensor goes back to the uploaded one."""
        check(self._lib.rk_restore(self._h))

    # RESCALk replicas ----------------------------------------------------------
    def tensor_export(self) -> bytes:
        """IPC record of this engine's uploaded dense tensor (rank 0 of a replica set)."""
        buf = ctypes.create_string_buffer(256)
        check(self._lib.rk_tensor_export(self._h, buf, 256))
        return buf.raw

    def tensor_import(self, record: bytes):
        """Copy an exported tensor peer-to-peer (NVLink) into this engine."""
        buf = ctypes.create_string_buffer(bytes(record), 256)
        check(self._lib.rk_tensor_import(self._h, buf))

    # p_r x p_c grid ------------------------------------------------------------
    def grid_init(self, pr, pc, rank, nccl_id: bytes):
        buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        check(self._lib.rk_grid_init(self._h, int(pr), int(pc), int(rank), buf, self.n))

    def grid_block(self):
        out = np.zeros(8, dtype=np.int64)
        check(self._lib.rk_grid_block(self._h, out.ctypes.data_as(_pi64), 8))
        keys = ["gi", "gj", "piece", "rows", "cols", "row0", "pr", "pc"]
        info = dict(zip(keys, (int(v) for v in out)))
        cm = np.zeros(info["cols"], dtype=np.int64)
        check(self._lib.rk_grid_colmap(self._h, cm.ctypes.data_as(_pi64)))
        info["colmap"] = cm
        return info

    def timing(self):
        out = np.zeros(4, dtype=np.float64)
        check(self._lib.rk_last_timing(self._h, _dp(out), 4))
        return {"run_ms": out[0], "k1_ms": out[1], "k1_launches": int(out[2]), "launches": int(out[3])}

    def phase_timing(self):
        """ms per iteration of each phase of the last profiled rk_run:
        K1, K5+K2a, grid all-reduce, K2f, K2b/numerator(+RS), A update/gather."""
        out = np.zeros(6, dtype=np.float64)
        check(self._lib.rk_phase_timing(self._h, _dp(out), 6))
        names = ["k1", "k2a", "allreduce", "k2f", "numer_rs", "apply_gather"]
        return dict(zip(names, out.tolist()))

    def time_k1(self, reps=10):
        ms = _f64(0.0)
        check(self._lib.rk_time_k1(self._h, int(reps), ctypes.byref(ms)))
        return ms.value

    def info(self):
        out = np.zeros(14, dtype=np.int64)
        check(self._lib.rk_info(self._h, out.ctypes.data_as(_pi64), 14))
        keys = ["engine", "n_pad", "k_pad", "strip_tiles", "ctas", "smem", "strips", "slots", "k2a_blocks", "nc_pad",
                "peer_exchange", "k1_merge_q", "k1_group", "strip_width"]
        return dict(zip(keys, (int(v) for v in out)))

    @property
    def stream(self):
        return self._lib.rk_stream(self._h)


def device_count():
    n = _i32(0)
    check(load().rk_device_count(ctypes.byref(n)))
    return n.value


def pcg64_draws(entropy, offset, count):
    """Device PCG64 draws u_{offset..offset+count} (tests / parity checks)."""
    sh, sl, ih, il = pcg64_seed_state(entropy)
    out = np.empty(count, dtype=np.float64)
    check(load().rk_pcg64_draws(sh, sl, ih, il, int(offset), int(count), _dp(out)))
    return out


def pcg64_random_on(device, entropy, count):
    """np.random.default_rng(SeedSequence(entropy)).random(count), bit for bit,
    drawn on `device` (PCG64 jump-ahead per thread) and copied back."""
    sh, sl, ih, il = pcg64_seed_state(entropy)
    out = np.empty(count, dtype=np.float64)
    check(load().rk_pcg64_draws_on(int(device), sh, sl, ih, il, 0, int(count), _dp(out)))
    return out


def perturb_values(entropy, delta, values: np.ndarray, e0: int = 0, field_only: bool = False, device: int = 0):
    """In place: values (contiguous f32/f64, the C-ordered elements e0..) times
    the PCG64 multiplier field of `entropy` (or the field itself)."""
    if values.dtype not in (np.float32, np.float64) or not values.flags.c_contiguous:
        raise DataError("perturb_values needs a C-contiguous float32/float64 array")
    sh, sl, ih, il = pcg64_seed_state(entropy)
    check(load().rk_perturb_values(int(device), sh, sl, ih, il, float(delta),
                                   RK_F32 if values.dtype == np.float32 else RK_F64,
                                   values.ctypes.data, int(values.size), int(e0), int(bool(field_only))))


def perturb_csr_values(entropy, delta, t: int, n: int, indptr, indices, values: np.ndarray, device: int = 0):
    """In place: stored values of CSR slice t resampled at (t*n + i)*n + j."""
    if values.dtype not in (np.float32, np.float64) or not values.flags.c_contiguous:
        raise DataError("perturb_csr_values needs a C-contiguous float32/float64 array")
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int32)
    sh, sl, ih, il = pcg64_seed_state(entropy)
    check(load().rk_perturb_csr_values(int(device), sh, sl, ih, il, float(delta),
                                       RK_F32 if values.dtype == np.float32 else RK_F64, int(t), int(n),
                                       ip.ctypes.data_as(_pi64), ix.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                       values.ctypes.data, int(values.size)))


def debug_guards(on: bool) -> None:
    """Guard bands after every later device allocation (diagnostics)."""
    check(load().rk_debug_guards(1 if on else 0))


def debug_check_guards():
    """(overwritten guard bytes, guarded blocks live) -- 0 damaged = no overrun."""
    bad, n = _i64(0), _i64(0)
    check(load().rk_debug_check_guards(ctypes.byref(bad), ctypes.byref(n)))
    return int(bad.value), int(n.value)


def release_cached_memory() -> None:
    """Return the library's cached device blocks to the driver."""
    load().rk_release_cached_memory()


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(load().rk_nccl_unique_id(buf))
    return buf.raw


def uniform_values(seed, offset, count):
    out = np.empty(count, dtype=np.float32)
    check(load().rk_uniform_values(int(seed), int(offset), int(count), out.ctypes.data_as(_pf)))
    return out
