/*
 * rescal_b200.h — C-ABI of the B200-native RESCAL multiplicative-update engine.
 *
 * This is the drop-in boundary for the reference's MU hot path. The reference
 * (rescalkit, pure Python) has no FFI of its own; its internal swap seam is
 * `_mu_iteration(x_ops, a_row, a_col, r, eps, hooks, counters)`
 * (pkg/src/rescalkit/rescal.py:114-146) driven by `rescal_solve`
 * (rescal.py:186-225). Each entry point below names the reference function
 * it replaces. Plain pointers and sizes only; the Python mirror of the
 * reference API (paper_2202_09512_b200/) binds these with ctypes, and
 * INTEGRATION.md shows the binding a rescalkit maintainer would add.
 *
 * Conventions
 *   - Every call returns an rk_status; on failure rk_last_error() returns a
 *     thread-local message. Status classes map 1:1 onto the reference's
 *     exception hierarchy (errors.py:4-21): DATA -> DataError,
 *     NUMERICAL -> NumericalError, GRID -> GridError, DEVICE -> a CUDA/NCCL
 *     failure (no reference equivalent; raised as RescalkitError).
 *   - Host buffers are BORROWED for the duration of a call (copied to/from
 *     the device). Device buffers are OWNED by the handle and released by
 *     rk_destroy. A handle is bound to one device and one host thread.
 *   - Factors cross the boundary as float64 (row-major A (n,k), R (m,k,k)),
 *     whatever the tensor dtype; the Python layer casts to x.dtype the way
 *     rescal.py:205-209 does.
 */
#ifndef RESCAL_B200_H
#define RESCAL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RK_OK = 0,
  RK_ERR_DATA = 1,      /* DataError      (errors.py:8)  */
  RK_ERR_NUMERICAL = 2, /* NumericalError (errors.py:12) */
  RK_ERR_GRID = 3,      /* GridError      (errors.py:16) */
  RK_ERR_DEVICE = 4     /* CUDA / NCCL failure           */
} rk_status;

typedef enum { RK_F32 = 0, RK_F64 = 1 } rk_dtype;

typedef enum {
  RK_ENGINE_AUTO = 0, /* tcgen05 when k fits TMEM, else SIMT            */
  RK_ENGINE_TC = 1,   /* tcgen05 3xBF16 split-precision slice contraction */
  RK_ENGINE_SIMT = 2  /* CUDA-core fp32 slice contraction (large k)       */
} rk_engine;

typedef struct rk_handle rk_handle;

/* Library identification / last error (thread-local). */
int rk_version(void);
const char* rk_last_error(void);
int rk_device_count(int* out);

/* Create an engine for a dense tensor with m slices of n x n, rank k.
 * Replaces the setup half of rescal_solve (rescal.py:194-209). The tensor is
 * stored on the device as two bf16 planes (hi, lo) per element, zero padded
 * to a multiple of 128; k is padded to a multiple of 16 (exact: zero factor
 * entries stay zero under MU, rescal.py:144 / dist_rescal.py:15-16). */
int rk_create(int device, int64_t n, int64_t m, int32_t k, int32_t engine, rk_handle** out);
void rk_destroy(rk_handle* h);

/* Sparse tensor engine (cfg4 path): m CSR slices of n x n, rank k <= 32.
 * Replaces the SparseRelTensor operand path (tensor.py:86-139; scipy CSR
 * X_t @ A and X_t.T @ (A R_t) inside rescal.py:128,134-135). */
int rk_create_sparse(int device, int64_t n, int64_t m, int32_t k, rk_handle** out);

/* All slices at once: indptr is (m, n+1) int64 GLOBAL offsets into the
 * concatenated indices (int32 column ids, sorted per row, no duplicates —
 * the SparseRelTensor canonical form, tensor.py:96-104) and data (dtype).
 * The CSC (transposed) index arrays are built on the device. */
int rk_upload_csr(rk_handle* h, const int64_t* indptr, const int32_t* indices, const void* data,
                  int32_t dtype, int64_t nnz);

/* Per-slice form (no host-side concatenation): for t < m, indptrs[t] is the
 * slice's own (n+1) int64 indptr starting at 0, indices[t] / data[t] its
 * nnz_per_slice[t] column ids and values — i.e. the arrays of each canonical
 * scipy csr_matrix in SparseRelTensor.slices (tensor.py:86-104). Pageable
 * buffers stream through a pinned ring; validation (non-negative values,
 * column range: tensor.py:102-103) and ||X||^2 (rescal.py:160-165) run on
 * the device. */
int rk_upload_csr_slices(rk_handle* h, const int64_t* const* indptrs, const int32_t* const* indices,
                         const void* const* data, const int64_t* nnz_per_slice, int32_t dtype);

/* Host tensor -> device. x is (m, n, n) C-contiguous in `dtype`. Replaces the
 * dense RelTensor.slice_ops() operand view (tensor.py:67-69). Also records
 * ||X||^2 in fp64 from the host values (rescal.py:160-165). */
int rk_upload_dense(rk_handle* h, const void* x, int32_t dtype);

/* Same, but for one rank's block of a p_r x p_c grid: x is (m, rows, cols)
 * C-contiguous and lands in the top-left corner of the padded slices.
 * sq_norm_global: ||X||^2 of the whole tensor, or < 0 to have the ranks sum
 * the exact squares of their uploaded blocks on the device (all-reduced over
 * the grid; the blocks partition X). Collective when < 0. Replaces
 * dist_rescal.py:138-140 (_global_sum of _local_sq_norm). */
int rk_upload_block(rk_handle* h, const void* x, int32_t dtype, int64_t rows, int64_t cols,
                    double sq_norm_global);

/* Synthetic device-resident input (benchmarks): x = uniform [0,1) drawn with
 * a counter-based hash of (seed, t, i, j), rounded to fp32. */
int rk_fill_uniform(rk_handle* h, uint64_t seed);

/* Factors in/out (fp64, unpadded). Replaces the `initial` copy-in
 * (rescal.py:198-201) and the RescalFactors return (rescal.py:225). */
int rk_set_factors(rk_handle* h, const double* A, const double* R);
int rk_get_factors(rk_handle* h, double* A, double* R);

/* Run up to `iters` MU iterations (rescal.py:215-224 loop around
 * _mu_iteration, rescal.py:114-146). track_error!=0 writes the relative error
 * after each iteration into trace_out[0..*iters_done) (rescal.py:218-222);
 * tol<0 means no tolerance; the loop stops as soon as err < tol
 * (rescal.py:223-224). Non-finite factors -> RK_ERR_NUMERICAL
 * (rescal.py:168-170,217,220-221). */
int rk_run(rk_handle* h, int32_t iters, double eps, int32_t track_error, double tol,
           double* trace_out, int32_t* iters_done);

/* Split API: update_r (rescal.py:228-240) and update_a (rescal.py:243-258)
 * applied to the factors held by the handle. */
int rk_update_r(rk_handle* h, double eps);
int rk_update_a(rk_handle* h, double eps);

/* sum_t ||X_t - A R_t A^T||^2 (direct, rescal.py:149-157) and ||X||^2 for the
 * factors held by the handle; rel_error = sqrt(res/norm) (rescal.py:269-276). */
int rk_residual(rk_handle* h, double* sq_residual, double* sq_norm);

/* regress_r (rescal.py:293-324): with A fixed (the handle's A), fit R from
 * all-ones cores; result is left in the handle (read with rk_get_factors). */
int rk_regress_r(rk_handle* h, int32_t max_iters, double tol, double eps, int32_t* iters_done);

/* Multiply the device tensor by the RESCALk resampling field
 * 1 + delta*(2u-1), u = PCG64 doubles (dist_rescal.py:164-171,205-215).
 * (state_hi, state_lo, inc_hi, inc_lo) is numpy's PCG64 state after seeding
 * from SeedSequence((base_seed, 3, q)); element e = t*n*n + i*n + j consumes
 * draw e. The original tensor is kept; rk_perturb always starts from it.
 * row0/col0 and n_global locate a grid block inside the global tensor. */
int rk_perturb(rk_handle* h, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
               uint64_t inc_lo, double delta, int64_t n_global, int64_t row0, int64_t col0,
               const int64_t* col_map);

/* Host-format resampling, the reference's perturb() / perturbation_field()
 * (dist_rescal.py:164-171,205-215): `values` (dtype, host, in/out) are the
 * elements e0 .. e0+count-1 of the C-ordered (m, n, n) tensor; each becomes
 * value * (dtype)(1 + delta (2u_e - 1)), or the multiplier itself when
 * field_only, with u_e the e-th draw of numpy PCG64 seeded as (state, inc).
 * Bit-exact with the reference (fp64 field, cast, product in dtype). */
int rk_perturb_values(int32_t device, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                      double delta, int32_t dtype, void* values, int64_t count, uint64_t e0, int32_t field_only);

/* Sparse perturb(): the stored values of CSR slice t (indptr starting at 0,
 * n rows) are resampled at their elements (t*n + i)*n + j. */
int rk_perturb_csr_values(int32_t device, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                          double delta, int32_t dtype, int64_t t, int64_t n, const int64_t* indptr,
                          const int32_t* indices, void* values, int64_t nnz);

/* Tensor-file ingest (host only, no GPU needed), csrc/ingest.cpp: parse a
 * `%rescalk-coo` text file (replaces tensor.py:260-300 _load_sparse, a
 * pure-Python line loop) into canonical per-slice CSR arrays (tensor.py:96-104
 * canonical form: duplicates summed, columns sorted, zeros dropped) with the
 * reference's validation rules and error texts. rk_coo_open returns
 * RK_ERR_DATA with rk_coo_last_error() on malformed input; then for each
 * slice t: rk_coo_slice_nnz(h, t) entries, rk_coo_fill copies indptr (n+1,
 * starting at 0), column ids and fp64 values. */
typedef struct rk_coo rk_coo;
int rk_coo_open(const char* path, rk_coo** out, int64_t* n, int64_t* m, int64_t* nnz);
const char* rk_coo_last_error(void);
int64_t rk_coo_slice_nnz(const rk_coo* h, int64_t t);
int rk_coo_fill(const rk_coo* h, int64_t t, int64_t* indptr, int32_t* indices, double* data);
void rk_coo_close(rk_coo* h);

/* NNDSVD support (nndsvd_init, rescal.py:327-372): products with the
 * unfolding M = [X_1 .. X_m | X_1^T .. X_m^T] (n x 2nm) of the handle's
 * tensor, for a device subspace iteration in place of the reference's
 * LAPACK SVD / ARPACK svds of M (rescal.py:341-352). V, U, Y are n x b
 * row-major fp64; b <= 256 (dense) or b in {16, 32} (sparse).
 *   rk_gram_apply:        Y = M M^T V = sum_t X_t (X_t^T V) + X_t^T (X_t V)
 *   rk_unfold_sign_norms: per column c of M^T U, the squared norms of its
 *                         positive and negative parts (the yp / ym norms of
 *                         rescal.py:357-360 before the 1/s scaling)
 *   rk_positive_mean:     mean of the positive stored entries (rescal.py:375-383) */
int rk_gram_apply(rk_handle* h, const double* V, int32_t b, double* Y);
int rk_unfold_sign_norms(rk_handle* h, const double* U, int32_t b, double* pos2, double* neg2);
int rk_positive_mean(rk_handle* h, double* mean);

/* Device buffers of destroyed handles are cached by the library for reuse
 * (a caching allocator: handle teardown and re-creation skip cudaFree /
 * cudaMalloc). This returns every cached block to the driver. */
void rk_release_cached_memory(void);

/* Diagnostics (the GPU pool has no compute-sanitizer): with guards on, every
 * device block allocated afterwards is followed by a 64 KB band of a fixed
 * byte pattern; rk_debug_check_guards reports how many band bytes of live
 * and already-freed guarded blocks were overwritten (0 = no out-of-bounds
 * write past any buffer end). Engine-private; no reference counterpart. */
int rk_debug_guards(int32_t on);
int rk_debug_check_guards(int64_t* damaged_bytes, int64_t* blocks_checked);
/* Positive control: allocate 1000 bytes, write nbytes past the end, free. */
int rk_debug_overrun(int64_t nbytes);
/* The slice products of the handle's last K1 pass (dense engines): P = X_t A
 * into P[m][n_pad][k_pad] and Q = X_t^T A into Q[m][n_pad][k_pad] (fp32, the
 * padded layout rk_info reports). Accuracy tests of the tensor-core pass. */
int rk_debug_read_pq(rk_handle* h, float* P, float* Q);

/* Raw PCG64 draws u_{offset} .. u_{offset+count-1} (tests of the generator). */
int rk_pcg64_draws(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, uint64_t offset,
                   int64_t count, double* out);

/* The same draws generated on `device` (the random start of rescal.py:173-183,
 * np.random.default_rng(SeedSequence(...)).random((n, k)): one host copy of the
 * result instead of a sequential host generator over n*k doubles). */
int rk_pcg64_draws_on(int32_t device, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                      uint64_t offset, int64_t count, double* out);

/* Multi-GPU p_r x p_c grid (dist_rescal.py:113-161 generalised to non-square
 * grids). nccl_id is a 128-byte ncclUniqueId broadcast by the caller. The
 * handle then holds the (m, n/p_r, n/p_c) block of rank (i, j); A pieces of
 * b = ceil(n/p) rows; rank (i,j) owns piece i*p_c+j. */
int rk_grid_init(rk_handle* h, int32_t pr, int32_t pc, int32_t rank, const void* nccl_id,
                 int64_t n_global);
int rk_nccl_unique_id(void* out128);

/* RESCALk ensembles spread over GPUs ("replicas", model_select.py:445-471 with
 * the members distributed; one process per GPU): rank 0 uploads the tensor and
 * rk_tensor_export writes a <= 256-byte record (CUDA IPC handles of the device
 * planes + norms) that the caller ships to the other ranks; rk_tensor_import
 * copies the planes peer-to-peer over NVLink instead of every rank uploading
 * the same tensor over the host links. The exporter must not perturb or free
 * its tensor until every importer returned. */
int rk_tensor_export(rk_handle* h, void* out, int32_t out_bytes);
int rk_tensor_import(rk_handle* h, const void* in);

/* Timing of the last rk_run (device time, CUDA events on the engine stream):
 * out[0]=total ms, out[1]=slice-contraction (K1) ms per launch averaged,
 * out[2]=number of K1 launches, out[3]=kernel launches total. */
int rk_last_timing(rk_handle* h, double* out, int32_t n_out);

/* Raw stream handle (cudaStream_t) for callers that time on it. */
void* rk_stream(rk_handle* h);

/* Engine introspection: out[0]=engine used, out[1]=n_pad, out[2]=k_pad,
 * out[3]=strip tiles (TC), out[4]=CTAs (TC), out[5]=smem bytes (TC), out[6]=strips,
 * out[7]=Q slots, out[8]=K2a blocks, out[9]=nc_pad, out[10]=1 when the grid exchange
 * runs over peer memory (NVLink IPC; set by the first grid rk_run), 0 for NCCL,
 * out[11]=1 when K1 merges Q's hi/lo operands, out[12]=CTAs per K1 strip group (1, 2, 4),
 * out[13]=column tiles per strip (TC). */
int rk_info(rk_handle* h, int64_t* out, int32_t n_out);

#ifdef __cplusplus
}
#endif

#endif /* RESCAL_B200_H */
