// Sparse-X MU path: CSR / CSC SpMM kernels.
//
// Reference: the sparse branch of _mu_iteration — scipy CSR X_t @ A
// (rescal.py:128) and X_t.T @ (A R_t) via the implicit CSC view (:134-135),
// i.e. scipy sparsetools csr_matvecs (single-threaded C++).
//
// Storage (device, per handle): all slices concatenated —
//   csr_ptr int64 [M][n+1] (global offsets), csr_idx int32 [nnz], csr_val f32 [nnz]
//   csc_* the same for X_t^T, built on the device with a stable radix sort of
//   (col, row) keys (CSC indices sorted within each column = scipy's tocsc()).
// Work per iteration (restructured):
//   SP1  CSR pass:  P_t = X_t A           (rows; A rows gathered from L2)
//   K2a/K2f         G, S_t = A^T P_t, core update, trace (dense kernels)
//   SP2  CSC pass:  z_j = X_t[:, j]^T A on the fly,
//                   num_j = sum_t P_t[j] R_t^T + z_j R_t   (fp64 across t)
//   SPA             A_j <- A_j * num_j / (A_j M + m eps) + operand copies
// A "lane group" of G = K/4 lanes owns one row (column) and holds its K
// accumulators as one float4 per lane; each nonzero gathers one 16-byte
// chunk per lane (a coalesced K*4-byte A row per group).
#pragma once

#include "rk_common.cuh"

namespace rk {
namespace sp {

// n = CSR rows of the (local) block; A32 = the gathered factor rows (the
// block's column set); P row stride Npad.
template <int K>
__global__ void __launch_bounds__(256) sp_csr_pass(const Ctl* __restrict__ ctl,
                                                   const int64_t* __restrict__ ptr,
                                                   const int* __restrict__ idx,
                                                   const float* __restrict__ val,
                                                   const float* __restrict__ A32,
                                                   float* __restrict__ P, int n, int Npad, int M,
                                                   int skip_if_stopped) {
  if (skip_if_stopped && ctl->stop) return;
  constexpr int G = K / 4;
  const int lane = threadIdx.x & 31;
  const int q = lane % G;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t total = (int64_t)M * n;
  for (int64_t task = group; task < total; task += ngroups) {
    const int t = (int)(task / n);
    const int i = (int)(task - (int64_t)t * n);
    const int64_t b = ptr[(int64_t)t * (n + 1) + i], e = ptr[(int64_t)t * (n + 1) + i + 1];
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t p = b;
    for (; p + 4 <= e; p += 4) {
      int j[4];
      float v[4];
      float4 a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        j[u] = __ldg(idx + p + u);
        v[u] = __ldg(val + p + u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = __ldg(reinterpret_cast<const float4*>(A32 + (size_t)j[u] * K) + q);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        y.x = fmaf(v[u], a[u].x, y.x);
        y.y = fmaf(v[u], a[u].y, y.y);
        y.z = fmaf(v[u], a[u].z, y.z);
        y.w = fmaf(v[u], a[u].w, y.w);
      }
    }
    for (; p < e; ++p) {
      const int j = __ldg(idx + p);
      const float v = __ldg(val + p);
      const float4 a = __ldg(reinterpret_cast<const float4*>(A32 + (size_t)j * K) + q);
      y.x = fmaf(v, a.x, y.x);
      y.y = fmaf(v, a.y, y.y);
      y.z = fmaf(v, a.z, y.z);
      y.w = fmaf(v, a.w, y.w);
    }
    reinterpret_cast<float4*>(P + ((size_t)t * Npad + i) * K)[q] = y;
  }
}

// CSC pass fused with the A numerator. W32 = [R_t^T ; R_t] for all slices in
// shared memory (fp32). Per (column j, slice t): z = X_t[:, j]^T A (gathered),
// p = P_t[j]; lane q of the group owns output columns 4q..4q+3 and needs the
// full p, z vectors: exchanged with group-local shuffles. With P == nullptr
// (grid blocks, where the P and Q sides live on different row sets) only the
// z R_t part is formed: U_J = sum_t z_t R_t. n = CSC columns of the block.
template <int K>
__global__ void __launch_bounds__(512) sp_csc_numer(const Ctl* __restrict__ ctl,
                                                    const int64_t* __restrict__ ptr,
                                                    const int* __restrict__ idx,
                                                    const float* __restrict__ val,
                                                    const float* __restrict__ A32,
                                                    const float* __restrict__ P,
                                                    const float* __restrict__ W32,
                                                    double* __restrict__ num, int n, int Npad,
                                                    int M) {
  if (ctl->stop) return;
  extern __shared__ float shw[];
  constexpr int G = K / 4;
  for (int e = threadIdx.x; e < M * 2 * K * K / 4; e += blockDim.x)
    reinterpret_cast<float4*>(shw)[e] = __ldg(reinterpret_cast<const float4*>(W32) + e);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int q = lane % G;
  const int gbase = lane - q;  // first lane of the group
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t g0 = group - lane / G;  // first group of this warp (warp-uniform loop bound)
  for (int64_t jw = g0; jw < n; jw += ngroups) {
    const int64_t j = jw + lane / G;
    const bool active = j < n;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    // software pipeline over slices: next slice's column bounds and P row are
    // loaded while the current slice's gathers are in flight
    int64_t nb = 0, ne = 0;
    float4 npv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (active) {
      nb = ptr[j];
      ne = ptr[j + 1];
      if (P) npv = __ldg(reinterpret_cast<const float4*>(P + (size_t)j * K) + q);
    }
    for (int t = 0; t < M; ++t) {
      const int64_t b = nb, e = ne;
      const float4 pv = npv;
      if (active && t + 1 < M) {
        nb = ptr[(int64_t)(t + 1) * (n + 1) + j];
        ne = ptr[(int64_t)(t + 1) * (n + 1) + j + 1];
        if (P) npv = __ldg(reinterpret_cast<const float4*>(P + ((size_t)(t + 1) * Npad + j) * K) + q);
      }
      float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      int64_t p = b;
      for (; p + 4 <= e; p += 4) {
        int ii[4];
        float v[4];
        float4 a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ii[u] = __ldg(idx + p + u);
          v[u] = __ldg(val + p + u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          a[u] = __ldg(reinterpret_cast<const float4*>(A32 + (size_t)ii[u] * K) + q);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          z.x = fmaf(v[u], a[u].x, z.x);
          z.y = fmaf(v[u], a[u].y, z.y);
          z.z = fmaf(v[u], a[u].z, z.z);
          z.w = fmaf(v[u], a[u].w, z.w);
        }
      }
      for (; p < e; ++p) {
        const int i = __ldg(idx + p);
        const float v = __ldg(val + p);
        const float4 a = __ldg(reinterpret_cast<const float4*>(A32 + (size_t)i * K) + q);
        z.x = fmaf(v, a.x, z.x);
        z.y = fmaf(v, a.y, z.y);
        z.z = fmaf(v, a.z, z.z);
        z.w = fmaf(v, a.w, z.w);
      }
      const float* WrT = shw + (size_t)t * 2 * K * K;  // [d][c] = R_t[c][d]
      const float* Wr = WrT + K * K;                   // [d][c] = R_t[d][c]
      float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int src = 0; src < G; ++src) {
        const float p0 = __shfl_sync(0xffffffffu, pv.x, gbase + src);
        const float p1 = __shfl_sync(0xffffffffu, pv.y, gbase + src);
        const float p2 = __shfl_sync(0xffffffffu, pv.z, gbase + src);
        const float p3 = __shfl_sync(0xffffffffu, pv.w, gbase + src);
        const float z0 = __shfl_sync(0xffffffffu, z.x, gbase + src);
        const float z1 = __shfl_sync(0xffffffffu, z.y, gbase + src);
        const float z2 = __shfl_sync(0xffffffffu, z.z, gbase + src);
        const float z3 = __shfl_sync(0xffffffffu, z.w, gbase + src);
        const float pp[4] = {p0, p1, p2, p3}, zz[4] = {z0, z1, z2, z3};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int d = src * 4 + u;
          const float4 wr = *reinterpret_cast<const float4*>(WrT + d * K + 4 * q);
          const float4 wq = *reinterpret_cast<const float4*>(Wr + d * K + 4 * q);
          s[0] = fmaf(pp[u], wr.x, fmaf(zz[u], wq.x, s[0]));
          s[1] = fmaf(pp[u], wr.y, fmaf(zz[u], wq.y, s[1]));
          s[2] = fmaf(pp[u], wr.z, fmaf(zz[u], wq.z, s[2]));
          s[3] = fmaf(pp[u], wr.w, fmaf(zz[u], wq.w, s[3]));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] += (double)s[u];
    }
    if (active) {
      double* out = num + (size_t)j * K + 4 * q;
#pragma unroll
      for (int u = 0; u < 4; ++u) out[u] = acc[u];
    }
  }
}

// A update from the numerator (separate launch: the CSC pass gathers the OLD
// A from every block, so A cannot change until it has finished). One thread
// per row reads the whole old row before writing it.
template <int K>
__global__ void __launch_bounds__(256) sp_apply_a(Ctl* __restrict__ ctl, double* __restrict__ A64,
                                                  float* __restrict__ A32,
                                                  const double* __restrict__ num,
                                                  const double* __restrict__ Mm, int n,
                                                  double eps_m) {
  if (ctl->stop) return;
  __shared__ double Ms[K * K];
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) Ms[e] = Mm[e];
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double a[K], out[K];
#pragma unroll
    for (int d = 0; d < K; ++d) a[d] = A64[(size_t)i * K + d];
    bool bad = false;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      double deno = eps_m;
#pragma unroll
      for (int d = 0; d < K; ++d) deno = fma(a[d], Ms[d * K + c], deno);
      out[c] = a[c] * num[(size_t)i * K + c] / deno;
      bad |= !isfinite(out[c]);
    }
    if (bad) {
      ctl->nonfinite = 1;
      ctl->stop = 1;
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
      A64[(size_t)i * K + c] = out[c];
      A32[(size_t)i * K + c] = (float)out[c];
    }
  }
}

// Resampling of the stored values (dist_rescal.py:208-214: sparse tensors keep
// their pattern, X' = X * field[t, row, col]). Works on CSR (major = row) and
// on CSC (major = column) arrays; each entry jumps the PCG64 stream to its
// element index (t*n + i)*n + j.
__global__ void __launch_bounds__(256) sp_perturb(const int64_t* __restrict__ ptr,
                                                  const int* __restrict__ idx,
                                                  const float* __restrict__ val0,
                                                  float* __restrict__ val, int nmajor, int M,
                                                  int col_major, u128 state, u128 inc,
                                                  double delta, int64_t n_global, int64_t row0,
                                                  const int64_t* __restrict__ colmap) {
  // one thread per (t, major index); entries of a major index are contiguous.
  // Local (row, col) -> global (row0 + row, colmap[col]) for grid blocks.
  const int64_t total = (int64_t)M * nmajor;
  for (int64_t task = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; task < total;
       task += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(task / nmajor), a = (int)(task - (int64_t)t * nmajor);
    const int64_t b = ptr[(int64_t)t * (nmajor + 1) + a], e = ptr[(int64_t)t * (nmajor + 1) + a + 1];
    for (int64_t p = b; p < e; ++p) {
      const int o = idx[p];
      const int64_t il = col_major ? o : a, jl = col_major ? a : o;
      const int64_t i = row0 + il, j = colmap ? colmap[jl] : jl;
      const uint64_t el = (uint64_t)(((int64_t)t * n_global + i) * n_global + j);
      u128 s = pcg_advance(state, inc, el);
      const double u = pcg_next_double(s, inc);
      const double f = 1.0 + delta * (2.0 * u - 1.0);
      val[p] = (float)((double)val0[p] * f);
    }
  }
}

// Residual-free helper: ||X||^2 of the stored values (fp64), per block.
__global__ void __launch_bounds__(256) sp_sq_norm(const float* __restrict__ val, int64_t nnz,
                                                  double* __restrict__ part) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = val[e];
    acc += v * v;
  }
  acc = warp_sum(acc);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    part[blockIdx.x] = s;
  }
}

// CSC construction helpers: keys = (col << 32) | row per stored entry of
// slice t, then a stable radix sort; counts per column -> exclusive scan.
__global__ void sp_make_keys(const int64_t* __restrict__ ptr, const int* __restrict__ idx, int n,
                             int64_t base, int64_t nnz, uint64_t* __restrict__ keys) {
  // one thread per row: rows are independent, entries of a row are contiguous
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int64_t b = ptr[i] - base, e = ptr[i + 1] - base;
    for (int64_t p = b; p < e; ++p) keys[p] = ((uint64_t)(uint32_t)idx[base + p] << 32) | (uint32_t)i;
  }
}

__global__ void sp_split_keys(const uint64_t* __restrict__ keys, int64_t nnz, int* __restrict__ rows,
                              int* __restrict__ counts) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[e];
    rows[e] = (int)(uint32_t)(k & 0xffffffffu);
    atomicAdd(counts + (int)(k >> 32), 1);  // integer counts: order-independent
  }
}

__global__ void sp_offsets(const int* __restrict__ counts, int n, int64_t base,
                           int64_t* __restrict__ out_ptr) {
  // single-block exclusive scan over n counts (n up to a few million; one pass)
  __shared__ int64_t carry;
  __shared__ int64_t wsum[32];
  if (threadIdx.x == 0) carry = base;
  __syncthreads();
  for (int i0 = 0; i0 < n; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    int64_t v = i < n ? counts[i] : 0;
    // block inclusive scan
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int64_t s = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      wsum[lane] = s;
    }
    __syncthreads();
    const int64_t incl = x + (w > 0 ? wsum[w - 1] : 0);
    if (i < n) out_ptr[i] = carry + incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) out_ptr[n] = carry;
}

// Synthetic uniform-random sparse slices (benchmarks): nnz_target random
// (row, col) keys per slice from a counter hash, sorted, duplicates dropped
// (= sum_duplicates; values are then drawn per unique entry), values U(0, 1].
__global__ void sp_gen_keys(uint64_t seed, int t, int64_t count, int n, uint64_t* __restrict__ keys) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = splitmix64(seed * 0x9E3779B97F4A7C15ull + ((uint64_t)t << 40) + (uint64_t)e);
    const uint64_t i = (r >> 32) % (uint64_t)n, j = (r & 0xffffffffu) % (uint64_t)n;
    keys[e] = (i << 32) | j;
  }
}

__global__ void sp_mark_unique(const uint64_t* __restrict__ keys, int64_t count, int* __restrict__ flag) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    flag[e] = (e == 0 || keys[e] != keys[e - 1]) ? 1 : 0;
}

// flag -> exclusive positions (scan done with cub), scatter unique keys into
// (indices, row counts) and draw the value of each unique entry.
// flag[e] = 1 for the first copy of a key that lies in the (grid) block:
// rows [row0, row0 + rows) and columns with col_local[j] >= 0 (all columns on
// one GPU: col_local == nullptr).
__global__ void sp_mark_unique_block(const uint64_t* __restrict__ keys, int64_t count, int64_t row0,
                                     int64_t rows, const int* __restrict__ col_local,
                                     int* __restrict__ flag) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[e];
    const int64_t i = (int64_t)(k >> 32), j = (int64_t)(k & 0xffffffffu);
    const bool first = e == 0 || k != keys[e - 1];
    const bool in = i >= row0 && i < row0 + rows && (!col_local || col_local[j] >= 0);
    flag[e] = (first && in) ? 1 : 0;
  }
}

__global__ void sp_scatter_unique(const uint64_t* __restrict__ keys, const int* __restrict__ flag,
                                  const int* __restrict__ pos, int64_t count, int64_t base,
                                  int* __restrict__ idx, float* __restrict__ val,
                                  int* __restrict__ row_counts, uint64_t seed, int t, int64_t row0,
                                  const int* __restrict__ col_local) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[e]) continue;
    const uint64_t k = keys[e];
    const int i = (int)(k >> 32), j = (int)(k & 0xffffffffu);
    const int64_t p = base + pos[e];
    idx[p] = col_local ? col_local[j] : j;
    const uint64_t r = splitmix64(seed ^ (k * 0xD1B54A32D192ED03ull) ^ ((uint64_t)t << 56));
    val[p] = 1.0f - (float)(r >> 40) * (1.0f / 16777216.0f);  // (0, 1]
    atomicAdd(row_counts + (i - row0), 1);
  }
}

}  // namespace sp
}  // namespace rk
