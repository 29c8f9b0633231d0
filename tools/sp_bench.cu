// Sparse gather-pass experiments (cfg4 shape: m=32, n=2^20, ~10.5 nnz/row, k=16).
// Standalone: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo
//   -I../paper_2202_09512_b200/csrc tools/sp_bench.cu -o tools/sp_bench
// Times variants of P_t = X_t A (CSR, A rows gathered) with CUDA events.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cstring>
#include <cuda_runtime.h>
#include "rk_kernels.cuh"
#include "sparse.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

using namespace rk;

// ---------------------------------------------------------------- generator
// per row: 10 or 11 random columns (sorted), values U(0,1]
__global__ void gen_counts(int n, int M, uint64_t seed, int* cnt, int poisson) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < (int64_t)n * M; r += (int64_t)gridDim.x * blockDim.x) {
    if (!poisson) { cnt[r] = 10 + ((splitmix64(seed + r) >> 40) % 100 < 49 ? 1 : 0); continue; }
    // Poisson(10.49) by inversion, capped at 31
    const double u = (double)(splitmix64(seed + r) >> 11) * (1.0 / 9007199254740992.0);
    double pk = exp(-10.49), cdf = pk; int k = 0;
    while (u > cdf && k < 31) { ++k; pk *= 10.49 / k; cdf += pk; }
    cnt[r] = k;
  }
}
__global__ void gen_rows(int n, int M, uint64_t seed, const int64_t* ptr, int* idx, float* val) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < (int64_t)n * M; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = ptr[r], e = ptr[r + 1];
    int c[32];
    int L = (int)(e - b);
    for (int u = 0; u < L; ++u) c[u] = (int)(splitmix64(seed * 31 + r * 17 + u) % (uint64_t)n);
    for (int u = 1; u < L; ++u) { int x = c[u]; int v = u - 1; while (v >= 0 && c[v] > x) { c[v + 1] = c[v]; --v; } c[v + 1] = x; }
    for (int u = 0; u < L; ++u) { idx[b + u] = c[u]; val[b + u] = 1.0f - (float)(splitmix64(seed ^ (b + u)) >> 40) * (1.0f / 16777216.0f); }
  }
}

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ uint64_t pol_first() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ int ld_stream_i(const int* a, uint64_t pol) { int v; asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol)); return v; }
__device__ __forceinline__ float ld_stream_f(const float* a, uint64_t pol) { float v; asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol)); return v; }
__device__ __forceinline__ int4 ld_stream_i4(const int* a, uint64_t pol) { int4 v; asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a), "l"(pol)); return v; }
__device__ __forceinline__ float4 ld_gather(const float* a, uint64_t pol) { float4 v; asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a), "l"(pol)); return v; }
__device__ __forceinline__ float4 ld_gather_plain(const float* a) { float4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a)); return v; }
__device__ __forceinline__ int ld_l1_i(const int* a, uint64_t pol) { int v; asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol)); return v; }
__device__ __forceinline__ float ld_l1_f(const float* a, uint64_t pol) { float v; asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol)); return v; }
__device__ __forceinline__ float4 ld_gather_l1(const float* a, uint64_t pol) { float4 v; asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a), "l"(pol)); return v; }
__device__ __forceinline__ void st_stream4(float* a, float4 v, uint64_t pol) { asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" :: "l"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)); }

// V1: hints. UNR gathers in flight per group. HINT: 0 none, 1 stream evict_first, 2 +A evict_last
template <int UNR, int HINT>
__global__ void __launch_bounds__(256) csr_v1(const int64_t* __restrict__ ptr, const int* __restrict__ idx,
                                              const float* __restrict__ val, const float* __restrict__ A32,
                                              float* __restrict__ P, int n, int M, int mask = -1) {
  constexpr int K = 16, G = 4;
  const uint64_t pf = pol_first(), pl = pol_last();
  const int q = threadIdx.x & 3;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t total = (int64_t)M * n;
  for (int64_t task = group; task < total; task += ngroups) {
    const int64_t b = ptr[task + task / n], e = ptr[task + task / n + 1];
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t p = b;
    for (; p + UNR <= e; p += UNR) {
      int j[UNR]; float v[UNR]; float4 a[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (HINT == 1 || HINT == 2) { j[u] = ld_stream_i(idx + p + u, pf); v[u] = ld_stream_f(val + p + u, pf); }
        else if (HINT >= 3) { j[u] = ld_l1_i(idx + p + u, pf); v[u] = ld_l1_f(val + p + u, pf); }
        else { j[u] = __ldg(idx + p + u); v[u] = __ldg(val + p + u); }
        j[u] &= mask;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) a[u] = HINT == 5 ? ld_gather_plain(A32 + (size_t)j[u] * K + 4 * q) : HINT == 6 ? ld_gather(A32 + (size_t)j[u] * K + 4 * q, pl) : HINT == 4 ? ld_gather_l1(A32 + (size_t)j[u] * K + 4 * q, pl) : HINT == 2 ? ld_gather(A32 + (size_t)j[u] * K + 4 * q, pl) : __ldg(reinterpret_cast<const float4*>(A32 + (size_t)j[u] * K) + q);
#pragma unroll
      for (int u = 0; u < UNR; ++u) { y.x = fmaf(v[u], a[u].x, y.x); y.y = fmaf(v[u], a[u].y, y.y); y.z = fmaf(v[u], a[u].z, y.z); y.w = fmaf(v[u], a[u].w, y.w); }
    }
    for (; p < e; ++p) {
      const int j = __ldg(idx + p) & mask; const float v = __ldg(val + p);
      const float4 a = HINT == 4 ? ld_gather_l1(A32 + (size_t)j * K + 4 * q, pl) : HINT == 2 ? ld_gather(A32 + (size_t)j * K + 4 * q, pl) : __ldg(reinterpret_cast<const float4*>(A32 + (size_t)j * K) + q);
      y.x = fmaf(v, a.x, y.x); y.y = fmaf(v, a.y, y.y); y.z = fmaf(v, a.z, y.z); y.w = fmaf(v, a.w, y.w);
    }
    const int t = (int)(task / n), i = (int)(task - (int64_t)t * n);
    float* dst = P + ((size_t)t * n + i) * K + 4 * q;
    if (HINT >= 1) st_stream4(dst, y, pf); else *reinterpret_cast<float4*>(dst) = y;
  }
}

// V5: group-cooperative idx/val loads (lane q loads entry p+q), branch-free tail.
template <int STEP>
__global__ void __launch_bounds__(256) csr_v5(const int64_t* __restrict__ ptr, const int* __restrict__ idx,
                                              const float* __restrict__ val, const float* __restrict__ A32,
                                              float* __restrict__ P, int n, int M) {
  constexpr int K = 16, G = 4;
  const int lane = threadIdx.x & 31, q = lane & 3, gb = lane & ~3;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t total = (int64_t)M * n;
  for (int64_t task = group; task < total; task += ngroups) {
    const int64_t b = ptr[task + task / n], e = ptr[task + task / n + 1];
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t p = b; p < e; p += STEP) {
      int jl[STEP / 4]; float vl[STEP / 4];
#pragma unroll
      for (int w = 0; w < STEP / 4; ++w) {
        const int64_t pp = p + 4 * w + q;
        jl[w] = pp < e ? __ldg(idx + pp) : 0;
        vl[w] = pp < e ? __ldg(val + pp) : 0.f;
      }
      float4 a[STEP]; float v[STEP];
#pragma unroll
      for (int u = 0; u < STEP; ++u) {
        const int j = __shfl_sync(0xFu << gb, jl[u / 4], gb + (u & 3));
        v[u] = __shfl_sync(0xFu << gb, vl[u / 4], gb + (u & 3));
        a[u] = __ldg(reinterpret_cast<const float4*>(A32 + (size_t)j * K) + q);
      }
#pragma unroll
      for (int u = 0; u < STEP; ++u) { y.x = fmaf(v[u], a[u].x, y.x); y.y = fmaf(v[u], a[u].y, y.y); y.z = fmaf(v[u], a[u].z, y.z); y.w = fmaf(v[u], a[u].w, y.w); }
    }
    const int t = (int)(task / n), i = (int)(task - (int64_t)t * n);
    *reinterpret_cast<float4*>(P + ((size_t)t * n + i) * K + 4 * q) = y;
  }
}

// V6: one CSR pass computes P (gathers A[j]) and Q (scatter-add v*A[i] into Q[j] with vector atomics)
__global__ void __launch_bounds__(256) csr_pq_atomic(const int64_t* __restrict__ ptr, const int* __restrict__ idx,
                                                     const float* __restrict__ val, const float* __restrict__ A32,
                                                     float* __restrict__ P, float* __restrict__ Q, int n, int M) {
  constexpr int K = 16, G = 4;
  const int q = threadIdx.x & 3;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t total = (int64_t)M * n;
  for (int64_t task = group; task < total; task += ngroups) {
    const int t = (int)(task / n), i = (int)(task - (int64_t)t * n);
    const int64_t b = ptr[task + t], e = ptr[task + t + 1];
    const float4 ai = __ldg(reinterpret_cast<const float4*>(A32 + (size_t)i * K) + q);
    float* Qt = Q + (size_t)t * n * K;
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t p = b;
    for (; p + 4 <= e; p += 4) {
      int j[4]; float v[4]; float4 a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { j[u] = __ldg(idx + p + u); v[u] = __ldg(val + p + u); }
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = __ldg(reinterpret_cast<const float4*>(A32 + (size_t)j[u] * K) + q);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        y.x = fmaf(v[u], a[u].x, y.x); y.y = fmaf(v[u], a[u].y, y.y); y.z = fmaf(v[u], a[u].z, y.z); y.w = fmaf(v[u], a[u].w, y.w);
        float* d = Qt + (size_t)j[u] * K + 4 * q;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(d), "f"(v[u] * ai.x), "f"(v[u] * ai.y), "f"(v[u] * ai.z), "f"(v[u] * ai.w) : "memory");
      }
    }
    for (; p < e; ++p) {
      const int j = __ldg(idx + p); const float v = __ldg(val + p);
      const float4 a = __ldg(reinterpret_cast<const float4*>(A32 + (size_t)j * K) + q);
      y.x = fmaf(v, a.x, y.x); y.y = fmaf(v, a.y, y.y); y.z = fmaf(v, a.z, y.z); y.w = fmaf(v, a.w, y.w);
      float* d = Qt + (size_t)j * K + 4 * q;
      asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(d), "f"(v * ai.x), "f"(v * ai.y), "f"(v * ai.z), "f"(v * ai.w) : "memory");
    }
    *reinterpret_cast<float4*>(P + ((size_t)t * n + i) * K + 4 * q) = y;
  }
}

// V7: group per row, predicated batches of B gathers (no serial tail), next row's bounds prefetched.
template <int B, int PF>
__global__ void __launch_bounds__(256) csr_v7(const int64_t* __restrict__ ptr, const int* __restrict__ idx,
                                              const float* __restrict__ val, const float* __restrict__ A32,
                                              float* __restrict__ P, int n, int M, int mask = -1) {
  constexpr int K = 16, G = 4;
  const int q = threadIdx.x & 3;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t total = (int64_t)M * n;
  int64_t task = group;
  int64_t nb = 0, ne = 0;
  if (task < total) { nb = ptr[task + task / n]; ne = ptr[task + task / n + 1]; }
  for (; task < total; task += ngroups) {
    const int64_t b = nb, e = ne;
    const int64_t nt = task + ngroups;
    if (PF && nt < total) { nb = ptr[nt + nt / n]; ne = ptr[nt + nt / n + 1]; }
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t p = b; p < e; p += B) {
      int j[B]; float v[B]; float4 a[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const bool ok = p + u < e;
        j[u] = ok ? (__ldg(idx + p + u) & mask) : -1;
        v[u] = ok ? __ldg(val + p + u) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < B; ++u) a[u] = j[u] >= 0 ? __ldg(reinterpret_cast<const float4*>(A32 + (size_t)j[u] * K) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < B; ++u) { y.x = fmaf(v[u], a[u].x, y.x); y.y = fmaf(v[u], a[u].y, y.y); y.z = fmaf(v[u], a[u].z, y.z); y.w = fmaf(v[u], a[u].w, y.w); }
    }
    if (!PF && nt < total) { nb = ptr[nt + nt / n]; ne = ptr[nt + nt / n + 1]; }
    const int t = (int)(task / n), i = (int)(task - (int64_t)t * n);
    *reinterpret_cast<float4*>(P + ((size_t)t * n + i) * K + 4 * q) = y;
  }
}

// V8: warp-cooperative: a warp owns 8 consecutive rows; their entries [ptr[r0], ptr[r0+8]) are
// staged in shared memory with coalesced loads, then group g runs row r0+g from smem with
// predicated batches of B gathers.
template <int B>
__global__ void __launch_bounds__(256) csr_v8(const int64_t* __restrict__ ptr, const int* __restrict__ idx,
                                              const float* __restrict__ val, const float* __restrict__ A32,
                                              float* __restrict__ P, int n, int M, int mask = -1) {
  constexpr int K = 16, CAP = 256;
  __shared__ int sj[8][CAP];
  __shared__ float sv[8][CAP];
  const int lane = threadIdx.x & 31, q = lane & 3, g = lane >> 2, w = threadIdx.x >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t total = (int64_t)M * n;  // n % 8 == 0
  for (int64_t task0 = warp * 8; task0 < total; task0 += nwarps * 8) {
    const int64_t off = task0 / n;
    const int64_t pv = lane <= 8 ? ptr[task0 + off + lane] : 0;
    const int64_t wb = __shfl_sync(0xffffffffu, pv, 0), we = __shfl_sync(0xffffffffu, pv, 8);
    const int64_t mb = __shfl_sync(0xffffffffu, pv, g), me = __shfl_sync(0xffffffffu, pv, g + 1);
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t c0 = wb; c0 < we; c0 += CAP) {
      const int cnt = (int)min((int64_t)CAP, we - c0);
      __syncwarp();
#pragma unroll 4
      for (int e = lane; e < cnt; e += 32) { sj[w][e] = __ldg(idx + c0 + e) & mask; sv[w][e] = __ldg(val + c0 + e); }
      __syncwarp();
      const int lo = (int)max((int64_t)0, mb - c0), hi = (int)min((int64_t)cnt, me - c0);
      for (int p = lo; p < hi; p += B) {
        float4 a[B]; float v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const bool ok = p + u < hi;
          const int j = ok ? sj[w][p + u] : 0;
          v[u] = ok ? sv[w][p + u] : 0.f;
          a[u] = ok ? __ldg(reinterpret_cast<const float4*>(A32 + (size_t)j * K) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < B; ++u) { y.x = fmaf(v[u], a[u].x, y.x); y.y = fmaf(v[u], a[u].y, y.y); y.z = fmaf(v[u], a[u].z, y.z); y.w = fmaf(v[u], a[u].w, y.w); }
      }
    }
    const int64_t task = task0 + g;
    const int t = (int)(task / n), i = (int)(task - (int64_t)t * n);
    *reinterpret_cast<float4*>(P + ((size_t)t * n + i) * K + 4 * q) = y;
  }
}

// V9: AoS records {idx, val} (8 B): one LDG.64 per entry (all 4 lanes of the group the same address).
template <int UNR>
__global__ void __launch_bounds__(256) csr_v9(const int64_t* __restrict__ ptr, const int2* __restrict__ rec,
                                              const float* __restrict__ A32, float* __restrict__ P, int n, int M, int mask = -1) {
  constexpr int K = 16, G = 4;
  const int q = threadIdx.x & 3;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t total = (int64_t)M * n;
  for (int64_t task = group; task < total; task += ngroups) {
    const int64_t b = ptr[task + task / n], e = ptr[task + task / n + 1];
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t p = b;
    for (; p + UNR <= e; p += UNR) {
      int2 r[UNR]; float4 a[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) r[u] = __ldg(rec + p + u);
#pragma unroll
      for (int u = 0; u < UNR; ++u) a[u] = __ldg(reinterpret_cast<const float4*>(A32 + (size_t)(r[u].x & mask) * K) + q);
#pragma unroll
      for (int u = 0; u < UNR; ++u) { const float v = __int_as_float(r[u].y); y.x = fmaf(v, a[u].x, y.x); y.y = fmaf(v, a[u].y, y.y); y.z = fmaf(v, a[u].z, y.z); y.w = fmaf(v, a[u].w, y.w); }
    }
    for (; p < e; ++p) {
      const int2 r = __ldg(rec + p);
      const float4 a = __ldg(reinterpret_cast<const float4*>(A32 + (size_t)(r.x & mask) * K) + q);
      const float v = __int_as_float(r.y);
      y.x = fmaf(v, a.x, y.x); y.y = fmaf(v, a.y, y.y); y.z = fmaf(v, a.z, y.z); y.w = fmaf(v, a.w, y.w);
    }
    const int t = (int)(task / n), i = (int)(task - (int64_t)t * n);
    *reinterpret_cast<float4*>(P + ((size_t)t * n + i) * K + 4 * q) = y;
  }
}

// V10: AoS, group-cooperative: lane q loads record p+q; (j, v) broadcast with shuffles; branch-free.
__global__ void __launch_bounds__(256) csr_v10(const int64_t* __restrict__ ptr, const int2* __restrict__ rec,
                                               const float* __restrict__ A32, float* __restrict__ P, int n, int M, int mask = -1) {
  constexpr int K = 16, G = 4;
  const int lane = threadIdx.x & 31, q = lane & 3, gb = lane & ~3;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t total = (int64_t)M * n;
  for (int64_t task = group; task < total; task += ngroups) {
    const int64_t b = ptr[task + task / n], e = ptr[task + task / n + 1];
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t p = b; p < e; p += 4) {
      const int2 r = p + q < e ? __ldg(rec + p + q) : make_int2(0, 0);
      float4 a[4]; float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = __shfl_sync(0xFu << gb, r.x, gb + u) & mask;
        v[u] = __int_as_float(__shfl_sync(0xFu << gb, r.y, gb + u));
        a[u] = __ldg(reinterpret_cast<const float4*>(A32 + (size_t)j * K) + q);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) { y.x = fmaf(v[u], a[u].x, y.x); y.y = fmaf(v[u], a[u].y, y.y); y.z = fmaf(v[u], a[u].z, y.z); y.w = fmaf(v[u], a[u].w, y.w); }
    }
    const int t = (int)(task / n), i = (int)(task - (int64_t)t * n);
    *reinterpret_cast<float4*>(P + ((size_t)t * n + i) * K + 4 * q) = y;
  }
}

__global__ void make_aos(const int* idx, const float* val, int64_t nnz, int2* rec) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    rec[e] = make_int2(idx[e], __float_as_int(val[e]));
}

// V11: V1 with column indices scaled into [0, rows) (table-size probe)
__global__ void __launch_bounds__(256) csr_v11(const int64_t* __restrict__ ptr, const int* __restrict__ idx,
                                               const float* __restrict__ val, const float* __restrict__ A32,
                                               float* __restrict__ P, int n, int M, int rows) {
  constexpr int K = 16, G = 4;
  const int q = threadIdx.x & 3;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t total = (int64_t)M * n;
  for (int64_t task = group; task < total; task += ngroups) {
    const int64_t b = ptr[task + task / n], e = ptr[task + task / n + 1];
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t p = b;
    for (; p + 4 <= e; p += 4) {
      int j[4]; float v[4]; float4 a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { j[u] = (int)(((uint64_t)__ldg(idx + p + u) * (uint64_t)rows) >> 20); v[u] = __ldg(val + p + u); }
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = __ldg(reinterpret_cast<const float4*>(A32 + (size_t)j[u] * K) + q);
#pragma unroll
      for (int u = 0; u < 4; ++u) { y.x = fmaf(v[u], a[u].x, y.x); y.y = fmaf(v[u], a[u].y, y.y); y.z = fmaf(v[u], a[u].z, y.z); y.w = fmaf(v[u], a[u].w, y.w); }
    }
    for (; p < e; ++p) {
      const int j = (int)(((uint64_t)__ldg(idx + p) * (uint64_t)rows) >> 20); const float v = __ldg(val + p);
      const float4 a = __ldg(reinterpret_cast<const float4*>(A32 + (size_t)j * K) + q);
      y.x = fmaf(v, a.x, y.x); y.y = fmaf(v, a.y, y.y); y.z = fmaf(v, a.z, y.z); y.w = fmaf(v, a.w, y.w);
    }
    const int t = (int)(task / n), i = (int)(task - (int64_t)t * n);
    *reinterpret_cast<float4*>(P + ((size_t)t * n + i) * K + 4 * q) = y;
  }
}

// V12: library kernel (hints, incremental task) + group-cooperative idx/val loads
template <int K>
__global__ void __launch_bounds__(256, 8) csr_v12(const int64_t* __restrict__ ptr, const int* __restrict__ idx,
                                                  const float* __restrict__ val, const float* __restrict__ A32,
                                                  float* __restrict__ P, int n, int Npad, int M) {
  constexpr int G = K / 4;
  const uint64_t pf = rk::sp::l2_evict_first(), pl = rk::sp::l2_evict_last();
  const int lane = threadIdx.x & 31;
  const int q = lane % G, gb = lane - q;
  const unsigned gmask = ((1u << G) - 1u) << gb;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int ngroups = (int)(((int64_t)gridDim.x * blockDim.x) / G);
  int t = (int)(group / n), i = (int)(group - (int64_t)t * n);
  for (; t < M;) {
    const int64_t* pt = ptr + (size_t)t * (n + 1);
    const int64_t b = pt[i], e = pt[i + 1];
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t p = b; p < e; p += G) {
      const bool ok = p + q < e;
      const int jq = ok ? rk::sp::ld_stream(idx + p + q, pf) : 0;
      const float vq = ok ? rk::sp::ld_stream(val + p + q, pf) : 0.f;
      float4 a[G];
      float v[G];
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int j = __shfl_sync(gmask, jq, gb + u);
        v[u] = __shfl_sync(gmask, vq, gb + u);
        a[u] = p + u < e ? rk::sp::ld_gather(A32 + (size_t)j * K + 4 * q, pl) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < G; ++u) {
        y.x = fmaf(v[u], a[u].x, y.x);
        y.y = fmaf(v[u], a[u].y, y.y);
        y.z = fmaf(v[u], a[u].z, y.z);
        y.w = fmaf(v[u], a[u].w, y.w);
      }
    }
    rk::sp::st_stream(P + ((size_t)t * Npad + i) * K + 4 * q, y, pf);
    i += ngroups;
    while (i >= n) { i -= n; ++t; }
  }
}

// S2: A chunk staged in smem, loop over slots; 4x4 register blocks, fp64 flush per 16 rows.
__global__ void __launch_bounds__(256) s_stream2(const float* __restrict__ A, const float* __restrict__ P, int n, int M,
                                                 int rows_per_chunk, double* __restrict__ part) {
  __shared__ float4 As[512 * 4];
  const int sub = threadIdx.x & 15, rl = threadIdx.x >> 4;
  const int c0 = (sub >> 2), d0 = (sub & 3);
  const int r0 = blockIdx.x * rows_per_chunk, r1 = min(n, r0 + rows_per_chunk);
  for (int base = r0; base < r1; base += 512) {
    const int nr = min(512, r1 - base);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * 4; e += 256) As[e] = __ldg(reinterpret_cast<const float4*>(A + (size_t)base * 16) + e);
    __syncthreads();
    for (int t = 0; t <= M; ++t) {
      const float* Pt = t < M ? P + (size_t)t * n * 16 : A;
      float s[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) s[u] = 0.f;
#pragma unroll 8
      for (int r = rl; r < nr; r += 16) {
        const float4 a = As[r * 4 + c0];
        const float4 p = __ldg(reinterpret_cast<const float4*>(Pt + (size_t)(base + r) * 16) + d0);
        const float av[4] = {a.x, a.y, a.z, a.w}, pv[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) s[x * 4 + y] = fmaf(av[x], pv[y], s[x * 4 + y]);
      }
      // 32 rows per thread per 512-row chunk: one fp64 write of the partial
      double* dst = part + (((size_t)t * gridDim.x + blockIdx.x) * 16 + rl) * 256 + sub * 16;
      if (base == r0) {
#pragma unroll
        for (int u = 0; u < 16; ++u) dst[u] = (double)s[u];
      } else {
#pragma unroll
        for (int u = 0; u < 16; ++u) dst[u] += (double)s[u];
      }
    }
  }
}

// V2: warp-cooperative rows. A warp owns 8 consecutive rows (one per group of 4 lanes);
// the warp loads the idx/val of its 8 rows cooperatively (coalesced) into registers via
// shuffles: nnz of the 8 rows are contiguous [ptr[r0], ptr[r0+8]).
template <int HINT>
__global__ void __launch_bounds__(256) csr_v2(const int64_t* __restrict__ ptr, const int* __restrict__ idx,
                                              const float* __restrict__ val, const float* __restrict__ A32,
                                              float* __restrict__ P, int n, int M) {
  constexpr int K = 16;
  const uint64_t pf = pol_first(), pl = pol_last();
  const int lane = threadIdx.x & 31, q = lane & 3, g = lane >> 2;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t total = (int64_t)M * n;  // n % 8 == 0
  for (int64_t task0 = warp * 8; task0 < total; task0 += nwarps * 8) {
    const int64_t task = task0 + g;
    const int64_t rowoff = task0 / n;  // slice index: ptr has n+1 entries per slice
    const int64_t myb = ptr[task + rowoff], mye = ptr[task + rowoff + 1];
    const int64_t wb = __shfl_sync(0xffffffffu, myb, 0);
    const int64_t we = __shfl_sync(0xffffffffu, mye, 28);
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t c0 = wb; c0 < we; c0 += 32) {
      // cooperative coalesced load of up to 32 entries
      int jj = 0; float vv = 0.f;
      if (c0 + lane < we) {
        if (HINT >= 1) { jj = ld_stream_i(idx + c0 + lane, pf); vv = ld_stream_f(val + c0 + lane, pf); }
        else { jj = __ldg(idx + c0 + lane); vv = __ldg(val + c0 + lane); }
      }
      // my row's entries within this chunk: [max(myb,c0), min(mye,c0+32))
      const int lo = (int)max((int64_t)0, myb - c0), hi = (int)min((int64_t)32, mye - c0);
      // iterate over the max count in the warp so shuffles stay converged
      int cnt = hi > lo ? hi - lo : 0;
      int maxcnt = cnt;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxcnt = max(maxcnt, __shfl_xor_sync(0xffffffffu, maxcnt, o));
      for (int u0 = 0; u0 < maxcnt; u0 += 4) {
        float4 a[4]; float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int src = min(lo + u0 + u, 31);
          const int j = __shfl_sync(0xffffffffu, jj, src);
          const float vx = __shfl_sync(0xffffffffu, vv, src);
          const bool ok = u0 + u < cnt;
          v[u] = ok ? vx : 0.f;
          const int jr = ok ? j : 0;
          a[u] = HINT >= 2 ? ld_gather(A32 + (size_t)jr * K + 4 * q, pl) : __ldg(reinterpret_cast<const float4*>(A32 + (size_t)jr * K) + q);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) { y.x = fmaf(v[u], a[u].x, y.x); y.y = fmaf(v[u], a[u].y, y.y); y.z = fmaf(v[u], a[u].z, y.z); y.w = fmaf(v[u], a[u].w, y.w); }
      }
    }
    const int t = (int)(task / n), i = (int)(task - (int64_t)t * n);
    float* dst = P + ((size_t)t * n + i) * K + 4 * q;
    if (HINT >= 1) st_stream4(dst, y, pf); else *reinterpret_cast<float4*>(dst) = y;
  }
}

// V3: half-k planes: A split into two [n][8] planes (32 B rows); HALF selects the plane.
template <int HINT>
__global__ void __launch_bounds__(256) csr_half(const int64_t* __restrict__ ptr, const int* __restrict__ idx,
                                                const float* __restrict__ val, const float* __restrict__ Ah,
                                                float* __restrict__ P, int n, int M, int half) {
  constexpr int G = 2;
  const uint64_t pf = pol_first(), pl = pol_last();
  const int q = threadIdx.x & 1;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t total = (int64_t)M * n;
  for (int64_t task = group; task < total; task += ngroups) {
    const int64_t b = ptr[task + task / n], e = ptr[task + task / n + 1];
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t p = b;
    for (; p + 4 <= e; p += 4) {
      int j[4]; float v[4]; float4 a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (HINT >= 1) { j[u] = ld_stream_i(idx + p + u, pf); v[u] = ld_stream_f(val + p + u, pf); }
        else { j[u] = __ldg(idx + p + u); v[u] = __ldg(val + p + u); }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = HINT >= 2 ? ld_gather(Ah + (size_t)j[u] * 8 + 4 * q, pl) : __ldg(reinterpret_cast<const float4*>(Ah + (size_t)j[u] * 8) + q);
#pragma unroll
      for (int u = 0; u < 4; ++u) { y.x = fmaf(v[u], a[u].x, y.x); y.y = fmaf(v[u], a[u].y, y.y); y.z = fmaf(v[u], a[u].z, y.z); y.w = fmaf(v[u], a[u].w, y.w); }
    }
    for (; p < e; ++p) {
      const int j = __ldg(idx + p); const float v = __ldg(val + p);
      const float4 a = __ldg(reinterpret_cast<const float4*>(Ah + (size_t)j * 8) + q);
      y.x = fmaf(v, a.x, y.x); y.y = fmaf(v, a.y, y.y); y.z = fmaf(v, a.z, y.z); y.w = fmaf(v, a.w, y.w);
    }
    const int t = (int)(task / n), i = (int)(task - (int64_t)t * n);
    float* dst = P + ((size_t)t * n + i) * 16 + 8 * half + 4 * q;
    if (HINT >= 1) st_stream4(dst, y, pf); else *reinterpret_cast<float4*>(dst) = y;
  }
}

// V4: gather ceiling: random 64 B (or 32 B) row gathers from a table of `rows` rows, no streams.
template <int ROWB>
__global__ void __launch_bounds__(256) gather_only(const float* __restrict__ A, int rows, int64_t count, float* out) {
  constexpr int G = ROWB / 16;
  const int q = threadIdx.x % G;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t e0 = group * 8; e0 < count; e0 += ngroups * 8) {
    float4 a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = (int)(splitmix64(e0 + u) % (uint64_t)rows);
      a[u] = __ldg(reinterpret_cast<const float4*>(A + (size_t)j * (ROWB / 4)) + q);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) { y.x += a[u].x; y.y += a[u].y; y.z += a[u].z; y.w += a[u].w; }
  }
  if (y.x == 123.f) out[0] = y.y + y.z + y.w;
}

// S_t = A^T P_t (fp32 products, fp64 flush every 16 rows). grid: (chunks, M+1); slot M = G (P := A)
__global__ void __launch_bounds__(256) s_stream(const float* __restrict__ A, const float* __restrict__ P, int n, int M,
                                                int rows_per_chunk, double* __restrict__ part) {
  // thread: 16 threads cover 16x16 with 4x4 blocks; 16 row-lanes per CTA
  const int t = blockIdx.y;
  const float* Pt = t < M ? P + (size_t)t * n * 16 : A;
  const int sub = threadIdx.x & 15, rl = threadIdx.x >> 4;  // rl: 0..15
  const int c0 = (sub >> 2) * 4, d0 = (sub & 3) * 4;
  const int r0 = blockIdx.x * rows_per_chunk, r1 = min(n, r0 + rows_per_chunk);
  double acc[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) acc[u] = 0.0;
  for (int rb = r0 + rl; rb < r1; rb += 16 * 16) {
    float s[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) s[u] = 0.f;
#pragma unroll 4
    for (int w = 0; w < 16; ++w) {
      const int r = rb + w * 16;
      if (r < r1) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(A + (size_t)r * 16 + c0));
        const float4 p = __ldg(reinterpret_cast<const float4*>(Pt + (size_t)r * 16 + d0));
        const float av[4] = {a.x, a.y, a.z, a.w}, pv[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) s[x * 4 + y] = fmaf(av[x], pv[y], s[x * 4 + y]);
      }
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) acc[u] += (double)s[u];
  }
  __shared__ double red[16][256];
#pragma unroll
  for (int u = 0; u < 16; ++u) red[rl][sub * 16 + u] = acc[u];
  __syncthreads();
  // 256 outputs (c,d) -> thread threadIdx.x sums the 16 row-lanes in order
  {
    const int o = threadIdx.x;  // o = sub*16 + u
    double s = 0.0;
    for (int l = 0; l < 16; ++l) s += red[l][o];
    const int sb = o >> 4, u = o & 15;
    const int c = (sb >> 2) * 4 + (u >> 2), d = (sb & 3) * 4 + (u & 3);
    part[((size_t)t * gridDim.x + blockIdx.x) * 256 + c * 16 + d] = s;
  }
}

// -------------------------------------------------------------------- main
template <class F>
float timeit(F f, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  CK(cudaGetLastError());
  return ms / reps;
}

int main(int argc, char** argv) {
  const int n = 1 << 20, M = 32, K = 16;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* cnt; int64_t* ptr; int* idx; float* val;
  CK(cudaMalloc(&cnt, sizeof(int) * (size_t)n * M));
  CK(cudaMalloc(&ptr, sizeof(int64_t) * ((size_t)n * M + 1)));
  const int poisson = getenv("POISSON") ? 1 : 0;
  gen_counts<<<sms * 8, 256>>>(n, M, 7, cnt, poisson);
  // exclusive scan on host (simple)
  std::vector<int> hc((size_t)n * M);
  CK(cudaMemcpy(hc.data(), cnt, hc.size() * 4, cudaMemcpyDeviceToHost));
  // ptr layout used by kernels: slice t row i -> ptr[t*(n+1) + i]; build that layout
  std::vector<int64_t> hp((size_t)(n + 1) * M);
  int64_t acc = 0;
  for (int t = 0; t < M; ++t) { for (int i = 0; i < n; ++i) { hp[(size_t)t * (n + 1) + i] = acc; acc += hc[(size_t)t * n + i]; } hp[(size_t)t * (n + 1) + n] = acc; }
  const int64_t nnz = acc;
  int64_t* ptr2; CK(cudaMalloc(&ptr2, sizeof(int64_t) * hp.size()));
  CK(cudaMemcpy(ptr2, hp.data(), hp.size() * 8, cudaMemcpyHostToDevice));
  // contiguous ptr for the generator (n*M+1)
  std::vector<int64_t> hp1((size_t)n * M + 1); acc = 0;
  for (size_t r = 0; r < (size_t)n * M; ++r) { hp1[r] = acc; acc += hc[r]; } hp1[(size_t)n * M] = acc;
  CK(cudaMemcpy(ptr, hp1.data(), hp1.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&idx, sizeof(int) * nnz)); CK(cudaMalloc(&val, sizeof(float) * nnz));
  gen_rows<<<sms * 8, 256>>>(n, M, 11, ptr, idx, val);
  CK(cudaDeviceSynchronize());
  printf("nnz=%lld (%.1f per row)\n", (long long)nnz, (double)nnz / ((double)n * M));
  float *A, *P, *Ah0, *Ah1, *out;
  CK(cudaMalloc(&A, sizeof(float) * n * K)); CK(cudaMalloc(&P, sizeof(float) * (size_t)n * K * M));
  CK(cudaMalloc(&Ah0, sizeof(float) * n * 8)); CK(cudaMalloc(&Ah1, sizeof(float) * n * 8)); CK(cudaMalloc(&out, 64));
  std::vector<float> ha((size_t)n * K);
  for (size_t e = 0; e < ha.size(); ++e) ha[e] = (float)((e * 2654435761u) % 1000) / 1000.f;
  CK(cudaMemcpy(A, ha.data(), ha.size() * 4, cudaMemcpyHostToDevice));
  std::vector<float> h0((size_t)n * 8), h1((size_t)n * 8);
  for (int i = 0; i < n; ++i) for (int c = 0; c < 8; ++c) { h0[(size_t)i * 8 + c] = ha[(size_t)i * 16 + c]; h1[(size_t)i * 8 + c] = ha[(size_t)i * 16 + 8 + c]; }
  CK(cudaMemcpy(Ah0, h0.data(), h0.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(Ah1, h1.data(), h1.size() * 4, cudaMemcpyHostToDevice));
  Ctl* ctl; CK(cudaMalloc(&ctl, sizeof(Ctl))); CK(cudaMemset(ctl, 0, sizeof(Ctl)));
  const double stream_gb = (8.0 * nnz + 8.0 * M * (n + 1) + 4.0 * n * K * M) / 1e9;
  const double gather_gb = 64.0 * nnz / 1e9;
  printf("algorithmic stream+P bytes %.2f GB, gather bytes %.2f GB\n", stream_gb, gather_gb);
  auto report = [&](const char* name, float ms) {
    printf("%-34s %8.3f ms  stream %6.0f GB/s  gather %6.0f GB/s\n", name, ms, stream_gb / ms * 1e3, gather_gb / ms * 1e3);
  };
  std::vector<float> ref((size_t)n * K * M), got((size_t)n * K * M);
  for (int gm : {8, 16, 32}) {
    if (argc > 1 && !strcmp(argv[1], "prof")) break;
    char nm[64]; snprintf(nm, 64, "V0 library grid=%d*sms", gm);
    report(nm, timeit([&] { sp::sp_csr_pass<16><<<sms * gm, 256>>>(ctl, ptr2, idx, val, A, P, n, n, M, 0); }));
  }
  CK(cudaMemcpy(ref.data(), P, ref.size() * 4, cudaMemcpyDeviceToHost));
  auto check = [&](const char* nm) {
    CK(cudaMemcpy(got.data(), P, got.size() * 4, cudaMemcpyDeviceToHost));
    double md = 0; for (size_t e = 0; e < got.size(); e += 97) md = std::max(md, (double)fabsf(got[e] - ref[e]));
    if (md > 1e-4) printf("   MISMATCH %s maxdiff %g\n", nm, md);
  };
  const char* which = argc > 1 ? argv[1] : "all";
  auto on = [&](const char* k) { return !strcmp(which, "all") || strstr(which, k); };
  if (on("mask")) for (int lg : {16, 18, 19, 20}) {
    char nm[64]; snprintf(nm, 64, "V1 unr4 cols masked to 2^%d", lg);
    report(nm, timeit([&] { csr_v1<4, 0><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M, (1 << lg) - 1); }));
  }
  if (on("coop2")) {
    report("V0 (hinted library)", timeit([&] { sp::sp_csr_pass<16><<<sms * 16, 256>>>(ctl, ptr2, idx, val, A, P, n, n, M, 0); }));
    report("V12 coop", timeit([&] { csr_v12<16><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, n, M); })); check("v12");
  }
  if (on("hint2")) {
    report("V1 unr4 hint0", timeit([&] { csr_v1<4, 0><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M); })); check("v1");
    report("V1 unr4 hint3 (stream L1+evict_first)", timeit([&] { csr_v1<4, 3><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M); })); check("v1");
    report("V1 unr4 hint5 (+gather L1 no_alloc)", timeit([&] { csr_v1<4, 5><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M); })); check("v1");
    report("V1 unr4 hint6 (+gather no_alloc evict_last)", timeit([&] { csr_v1<4, 6><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M); })); check("v1");
  }
  if (on("hint")) {
    report("V1 unr4 hint3 (stream L1+evict_first)", timeit([&] { csr_v1<4, 3><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M); })); check("v1");
    report("V1 unr4 hint4 (+A L1 evict_last)", timeit([&] { csr_v1<4, 4><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M); })); check("v1");
    report("V1 unr8 hint4", timeit([&] { csr_v1<8, 4><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M); })); check("v1");
  }
  if (on("coop")) {
    report("V5 coop step4", timeit([&] { csr_v5<4><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M); })); check("v5");
    report("V5 coop step8", timeit([&] { csr_v5<8><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M); })); check("v5");
    report("V5 coop step12", timeit([&] { csr_v5<12><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M); })); check("v5");
  }
  if (on("window")) {
    cudaStream_t st; cudaStreamCreate(&st);
    int maxp = 0; cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxp));
    for (float hr : {1.0f, 0.75f, 0.5f}) {
      cudaStreamAttrValue av{};
      av.accessPolicyWindow.base_ptr = A;
      av.accessPolicyWindow.num_bytes = (size_t)n * K * 4;
      av.accessPolicyWindow.hitRatio = hr;
      av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
      char nm[64]; snprintf(nm, 64, "V0 + persisting window hr=%.2f", hr);
      report(nm, timeit([&] { sp::sp_csr_pass<16><<<sms * 16, 256, 0, st>>>(ctl, ptr2, idx, val, A, P, n, n, M, 0); }));
      check("win");
      cudaCtxResetPersistingL2Cache();
    }
    cudaStreamAttrValue av{};
    av.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av);
  }
  // S stream
  double* part; const int chunks = sms * 2;
  CK(cudaMalloc(&part, sizeof(double) * (M + 1) * chunks * 256));
  if (!strcmp(which, "prof")) {
    csr_v1<4, 0><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M, (1 << 19) - 1);
    csr_v8<8><<<sms * 8, 256>>>(ptr2, idx, val, A, P, n, M, (1 << 19) - 1);
    csr_v1<4, 0><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M, -1);
    CK(cudaDeviceSynchronize());
    printf("prof done\n");
    return 0;
  }
  if (on("tsize")) {
    for (int rows : {1 << 19, 640 << 10, 704 << 10, 768 << 10, 832 << 10, 896 << 10, 1 << 20}) {
      char nm[64]; snprintf(nm, 64, "V1 table %d MB", rows * 64 >> 20);
      report(nm, timeit([&] { csr_v11<<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M, rows); }));
    }
  }
  if (on("aos")) {
    int2* rec; CK(cudaMalloc(&rec, sizeof(int2) * nnz));
    make_aos<<<sms * 8, 256>>>(idx, val, nnz, rec);
    for (int mk : {(1 << 19) - 1, -1}) {
      printf("-- mask %d\n", mk);
      report("V1 (ref)", timeit([&] { csr_v1<4, 0><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M, mk); }));
      report("V9 AoS unr4", timeit([&] { csr_v9<4><<<sms * 16, 256>>>(ptr2, rec, A, P, n, M, mk); })); if (mk == -1) check("v9");
      report("V9 AoS unr2", timeit([&] { csr_v9<2><<<sms * 16, 256>>>(ptr2, rec, A, P, n, M, mk); })); if (mk == -1) check("v9");
      report("V9 AoS unr6", timeit([&] { csr_v9<6><<<sms * 16, 256>>>(ptr2, rec, A, P, n, M, mk); })); if (mk == -1) check("v9");
      report("V5 coop8 (fixed mask)", timeit([&] { csr_v5<8><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M); })); if (mk == -1) check("v5");
      report("V10 AoS coop4", timeit([&] { csr_v10<<<sms * 16, 256>>>(ptr2, rec, A, P, n, M, mk); })); if (mk == -1) check("v10");
    }
    cudaFree(rec);
  }
  if (on("v7")) {
    for (int mk : {(1 << 19) - 1, -1}) {
      printf("-- mask %d\n", mk);
      report("V7 B=4 pf", timeit([&] { csr_v7<4, 1><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M, mk); })); if (mk == -1) check("v7");
      report("V7 B=8 pf", timeit([&] { csr_v7<8, 1><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M, mk); })); if (mk == -1) check("v7");
      report("V7 B=8 nopf", timeit([&] { csr_v7<8, 0><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M, mk); })); if (mk == -1) check("v7");
      report("V7 B=12 pf", timeit([&] { csr_v7<12, 1><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M, mk); })); if (mk == -1) check("v7");
      report("V7 B=16 pf", timeit([&] { csr_v7<16, 1><<<sms * 16, 256>>>(ptr2, idx, val, A, P, n, M, mk); })); if (mk == -1) check("v7");
      report("V8 B=4", timeit([&] { csr_v8<4><<<sms * 8, 256>>>(ptr2, idx, val, A, P, n, M, mk); })); if (mk == -1) check("v8");
      report("V8 B=8", timeit([&] { csr_v8<8><<<sms * 8, 256>>>(ptr2, idx, val, A, P, n, M, mk); })); if (mk == -1) check("v8");
      report("V8 B=12", timeit([&] { csr_v8<12><<<sms * 8, 256>>>(ptr2, idx, val, A, P, n, M, mk); })); if (mk == -1) check("v8");
    }
  }
  if (on("atomic")) {
    float* Q; CK(cudaMalloc(&Q, sizeof(float) * (size_t)n * K * M));
    float ms = timeit([&] { cudaMemsetAsync(Q, 0, sizeof(float) * (size_t)n * K * M); csr_pq_atomic<<<sms * 16, 256>>>(ptr2, idx, val, A, P, Q, n, M); });
    report("V6 P + Q-scatter atomics (+memset)", ms); check("v6");
    ms = timeit([&] { cudaMemsetAsync(Q, 0, sizeof(float) * (size_t)n * K * M); });
    printf("   (memset Q alone %.3f ms)\n", ms);
    cudaFree(Q);
  }
  if (on("k2b")) {
    float *Q, *W32; double *A64, *Mm; __nv_bfloat16 *ATh, *ATl;
    CK(cudaMalloc(&Q, sizeof(float) * (size_t)n * K * M)); CK(cudaMemcpy(Q, P, sizeof(float) * (size_t)n * K * M, cudaMemcpyDeviceToDevice));
    CK(cudaMalloc(&W32, sizeof(float) * M * 2 * K * K)); CK(cudaMemset(W32, 0, sizeof(float) * M * 2 * K * K));
    CK(cudaMalloc(&A64, sizeof(double) * n * K)); CK(cudaMemset(A64, 0, sizeof(double) * n * K));
    CK(cudaMalloc(&Mm, sizeof(double) * K * K)); CK(cudaMemset(Mm, 0, sizeof(double) * K * K));
    CK(cudaMalloc(&ATh, 2 * (size_t)n * K)); CK(cudaMalloc(&ATl, 2 * (size_t)n * K));
    float* A32b; CK(cudaMalloc(&A32b, sizeof(float) * n * K));
    for (int tg : {2, 4, 8}) {
      const int rb = 2 * (256 / K);
      const size_t smem = (size_t)tg * (2 * K * K + 2 * rb * K) * sizeof(float);
      CK(cudaFuncSetAttribute(k2b_v4<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      float ms = timeit([&] { k2b_v4<16><<<(n + rb - 1) / rb, 256, smem>>>(ctl, A64, A32b, ATh, ATl, P, Q, W32, Mm, n, M, tg, 1e-16); });
      printf("k2b_v4 tg=%d                        %8.3f ms  %6.0f GB/s (P+Q reads)\n", tg, ms, 8.0 * n * K * M / ms / 1e6);
    }
    {
      double* num; CK(cudaMalloc(&num, sizeof(double) * n * K));
      const size_t wsm = (size_t)M * 2 * K * K * sizeof(float);
      CK(cudaFuncSetAttribute(sp::sp_csc_numer<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
      for (int gm : {4, 8}) {
        float ms = timeit([&] { sp::sp_csc_numer<16><<<sms * gm / 2, 512, wsm>>>(ctl, ptr2, idx, val, A, P, W32, num, n, n, M); });
        printf("sp_csc_numer (P+z) grid=%d*sms/2    %8.3f ms\n", gm, ms);
        ms = timeit([&] { sp::sp_csc_numer<16><<<sms * gm / 2, 512, wsm>>>(ctl, ptr2, idx, val, A, nullptr, W32, num, n, n, M); });
        printf("sp_csc_numer (z only) grid=%d*sms/2 %8.3f ms\n", gm, ms);
      }
    }
    double* red; CK(cudaMalloc(&red, sizeof(double) * (M + 1) * K * K));
    for (int ncta : {8, 16}) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(ncta, (unsigned)(M + 1));
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = rk::k2a_v4_smem(K);
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = ncta; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr; cfg.numAttrs = 1;
      if (ncta == 16) CK(cudaFuncSetAttribute(k2a_v4<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      CK(cudaFuncSetAttribute(k2a_v4<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes));
      float ms = timeit([&] { CK(cudaLaunchKernelEx(&cfg, k2a_v4<16>, (const Ctl*)ctl, (const float*)A, (const float*)A, n, (const float*)P, n, M, red, 0)); });
      printf("k2a_v4 cluster=%d                   %8.3f ms  %6.0f GB/s (P reads)\n", ncta, ms, 4.0 * n * K * M / ms / 1e6);
    }
  }
  if (on("sstream")) {
    const int rpc = (n + chunks - 1) / chunks;
    float ms = timeit([&] { s_stream<<<dim3(chunks, M + 1), 256>>>(A, P, n, M, rpc, part); });
    printf("%-34s %8.3f ms  %6.0f GB/s (P+A reads)\n", "S_t = A^T P_t stream", ms, (4.0 * n * K * M + 4.0 * n * K * (M + 1)) / ms / 1e6);
    for (int ch : {sms * 2, sms * 4, sms * 8}) {
      double* part2; CK(cudaMalloc(&part2, sizeof(double) * (M + 1) * ch * 16 * 256));
      const int rpc2 = ((n + ch - 1) / ch + 511) / 512 * 512;
      const int chn = (n + rpc2 - 1) / rpc2;
      ms = timeit([&] { s_stream2<<<chn, 256>>>(A, P, n, M, rpc2, part2); });
      printf("S2 chunks=%d rpc=%d                %8.3f ms  %6.0f GB/s (P+A reads)\n", chn, rpc2, ms, (4.0 * n * K * M + 4.0 * n * K) / ms / 1e6);
      cudaFree(part2);
    }
  }
  return 0;
}
