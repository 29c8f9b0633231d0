// Gather-throughput experiment for the sparse passes (cfg4: 64 B factor rows,
// random row indices, 2^20-row table). Compares
//   ldg   : lane groups of 4 lanes, one LDG.128 per lane per row (current sp_csr_pass)
//   g4    : TMA tile::gather4 (4 rows per instruction) into a shared-memory ring,
//           consumer warps read the staged rows with LDS.128
//   bulk  : cp.async.bulk (non-tensor) 64 B per row into the same ring
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo tools/tma_gather_bench.cu -lcuda -o tools/tma_gather_bench
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint64_t smix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__global__ void gen_idx(int* idx, int64_t E, int rows) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    idx[e] = (int)(smix(e) % (uint64_t)rows);
}
__global__ void gen_tab(float* t, int64_t N) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x)
    t[e] = (float)(smix(e * 7 + 3) >> 40) * (1.0f / 16777216.0f);
}

__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_first() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }

// ---------------------------------------------------------------- ldg
__global__ void __launch_bounds__(256, 8) k_ldg(const int* __restrict__ idx, int64_t E, const float* __restrict__ tab, float* out) {
  const uint64_t pl = pol_last(), pf = pol_first();
  const int q = threadIdx.x & 3;
  const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 2;
  float4 y = make_float4(0, 0, 0, 0);
  for (int64_t e = g0 * 4; e < E; e += ng * 4) {
    int j[4];
    float4 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(j[u]) : "l"(idx + e + u), "l"(pf));
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                   : "=f"(a[u].x), "=f"(a[u].y), "=f"(a[u].z), "=f"(a[u].w)
                   : "l"(tab + (size_t)j[u] * 16 + 4 * q), "l"(pl));
#pragma unroll
    for (int u = 0; u < 4; ++u) { y.x += a[u].x; y.y += a[u].y; y.z += a[u].z; y.w += a[u].w; }
  }
  atomicAdd(out, y.x + y.y + y.z + y.w);
}


// LPR lanes per row, VEC floats per lane load (16 = LPR*VEC); ALLOC: 0 no_allocate, 1 L1 allocate
template <int LPR, int ALLOC>
__global__ void __launch_bounds__(256, 8) k_ldgv(const int* __restrict__ idx, int64_t E, const float* __restrict__ tab, float* out) {
  constexpr int VEC = 16 / LPR;
  const uint64_t pl = pol_last(), pf = pol_first();
  const int q = threadIdx.x % LPR;
  const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / LPR;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / LPR;
  float acc = 0.f;
  for (int64_t e = g0 * 4; e < E; e += ng * 4) {
    int j[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(j[u]) : "l"(idx + e + u), "l"(pf));
    float a[4][VEC];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float* src = tab + (size_t)j[u] * 16 + VEC * q;
      if constexpr (VEC == 16) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
          asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                       : "=f"(a[u][8*h+0]), "=f"(a[u][8*h+1]), "=f"(a[u][8*h+2]), "=f"(a[u][8*h+3]), "=f"(a[u][8*h+4]), "=f"(a[u][8*h+5]), "=f"(a[u][8*h+6]), "=f"(a[u][8*h+7])
                       : "l"(src + 8 * h), "l"(pl));
      } else if constexpr (VEC == 8) {
        if (ALLOC)
          asm volatile("ld.global.nc.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                       : "=f"(a[u][0]), "=f"(a[u][1]), "=f"(a[u][2]), "=f"(a[u][3]), "=f"(a[u][4]), "=f"(a[u][5]), "=f"(a[u][6]), "=f"(a[u][7])
                       : "l"(src), "l"(pl));
        else
          asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                       : "=f"(a[u][0]), "=f"(a[u][1]), "=f"(a[u][2]), "=f"(a[u][3]), "=f"(a[u][4]), "=f"(a[u][5]), "=f"(a[u][6]), "=f"(a[u][7])
                       : "l"(src), "l"(pl));
      } else if constexpr (VEC == 4) {
        if (ALLOC)
          asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                       : "=f"(a[u][0]), "=f"(a[u][1]), "=f"(a[u][2]), "=f"(a[u][3]) : "l"(src), "l"(pl));
        else
          asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                       : "=f"(a[u][0]), "=f"(a[u][1]), "=f"(a[u][2]), "=f"(a[u][3]) : "l"(src), "l"(pl));
      } else if constexpr (VEC == 2) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
                     : "=f"(a[u][0]), "=f"(a[u][1]) : "l"(src), "l"(pl));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int h = 0; h < VEC; ++h) acc += a[u][h];
  }
  atomicAdd(out, acc);
}
// one row per LDG: only lanes 0..3 of each warp active (rows per warp-instruction = 1)
__global__ void __launch_bounds__(256, 8) k_ldg1(const int* __restrict__ idx, int64_t E, const float* __restrict__ tab, float* out) {
  const uint64_t pl = pol_last();
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (int64_t e = w0 * 8; e < E; e += nw * 8) {
    const int jl = idx[e + (lane & 7)];
    float4 a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = __shfl_sync(0xffffffffu, jl, u);
      if (lane < 4)
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=f"(a[u].x), "=f"(a[u].y), "=f"(a[u].z), "=f"(a[u].w) : "l"(tab + (size_t)j * 16 + 4 * lane), "l"(pl));
      else a[u] = make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += a[u].x + a[u].y + a[u].z + a[u].w;
  }
  atomicAdd(out, acc);
}


// RPL distinct rows per warp-LDG.128 (lane groups of 4 lanes; groups beyond RPL
// duplicate the addresses of group (g % RPL)); 16 rows per warp iteration.
template <int RPL>
__global__ void __launch_bounds__(256, 4) k_rpl(const int* __restrict__ idx, int64_t E, const float* __restrict__ tab, float* out) {
  const uint64_t pl = pol_last();
  const int lane = threadIdx.x & 31, q = lane & 3, g = (lane >> 2) % RPL;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  constexpr int NL = 16 / RPL;  // loads per lane per iteration
  for (int64_t e = w0 * 16; e < E; e += nw * 16) {
    const int jl = idx[e + (lane & 15)];
    float4 a[NL];
#pragma unroll
    for (int u = 0; u < NL; ++u) {
      const int j = __shfl_sync(0xffffffffu, jl, u * RPL + g);
      asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                   : "=f"(a[u].x), "=f"(a[u].y), "=f"(a[u].z), "=f"(a[u].w) : "l"(tab + (size_t)j * 16 + 4 * q), "l"(pl));
    }
#pragma unroll
    for (int u = 0; u < NL; ++u) { acc.x += a[u].x; acc.y += a[u].y; acc.z += a[u].z; acc.w += a[u].w; }
  }
  if ((lane >> 2) < RPL) atomicAdd(out, acc.x + acc.y + acc.z + acc.w);
}

// ---------------------------------------------------------------- mbarrier helpers
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(sa(b)), "r"(ph)
      : "memory");
}

constexpr int RS = 128;       // rows per stage
constexpr int NSTG = 16;      // stages
constexpr int NCW = 4;        // consumer warps

// MODE 0: gather4 tensor TMA, MODE 1: cp.async.bulk 64 B per row
template <int MODE>
__global__ void __launch_bounds__(32 * (NCW + 1), 1) k_tma(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                                           int64_t E, const float* __restrict__ tab, float* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);
  __shared__ uint64_t full[NSTG], empty[NSTG];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTG; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], NCW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nchunks = E / RS;
  float acc = 0.f;
  if (warp == 0) {
    const uint64_t pf = pol_first(), pl = pol_last();
    int s = 0; uint32_t ph = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      mb_wait(&empty[s], ph ^ 1);
      int4 j;
      asm volatile("ld.global.nc.L2::cache_hint.v4.b32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(j.x), "=r"(j.y), "=r"(j.z), "=r"(j.w) : "l"(idx + c * RS + 4 * lane), "l"(pf));
      if (lane == 0) mb_expect(&full[s], RS * 64);
      __syncwarp();
      const uint32_t dst = sa(ring + ((size_t)s * RS + 4 * lane) * 16);
      if (MODE == 0) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
            "l"(&tm), "r"(0), "r"(j.x), "r"(j.y), "r"(j.z), "r"(j.w), "r"(sa(&full[s])), "l"(pl)
            : "memory");
      } else {
        const int jj[4] = {j.x, j.y, j.z, j.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], 64, [%2], %3;" ::"r"(dst + 64 * u),
                       "l"(tab + (size_t)jj[u] * 16), "r"(sa(&full[s])), "l"(pl)
                       : "memory");
      }
      if (++s == NSTG) { s = 0; ph ^= 1; }
    }
  } else {
    const int cw = warp - 1;
    int s = 0; uint32_t ph = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      mb_wait(&full[s], ph);
      // this warp's 32 rows = 2 KB: 4 float4 per lane
      const float4* r = reinterpret_cast<const float4*>(ring + ((size_t)s * RS + cw * 32) * 16);
#pragma unroll
      for (int u = 0; u < 4; ++u) { float4 v = r[u * 32 + lane]; acc += v.x + v.y + v.z + v.w; }
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[s]);
      if (++s == NSTG) { s = 0; ph ^= 1; }
    }
  }
  atomicAdd(out, acc);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int64_t E = 1ll << 27;  // 134M gathers (8.6 GB of rows)
  int* idx; float* tab; float* out;
  CK(cudaMalloc(&idx, E * 4));
  CK(cudaMalloc(&tab, (1ll << 20) * 64));
  CK(cudaMalloc(&out, 4));
  gen_tab<<<2048, 256>>>(tab, (1ll << 20) * 16);
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  void* p; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)p;
  const size_t smem = (size_t)NSTG * RS * 64;
  CK(cudaFuncSetAttribute(k_tma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int lg = 19; lg <= 20; ++lg) {
    const int rows = 1 << lg;
    gen_idx<<<4096, 256>>>(idx, E, rows);
    CUtensorMap tm;
    cuuint64_t dims[2] = {16, (cuuint64_t)rows};
    cuuint64_t strides[1] = {64};
    cuuint32_t box[2] = {16, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    const char* nm[] = {"ldg4x128", "ldg8x64", "ldg2x256", "ldg1x2x256", "ldg4x128_l1", "ldg2x256_l1", "ldg1row", "gather4", "rpl8", "rpl4", "rpl2", "rpl1"};
    for (int mode = 0; mode < 12; ++mode) {
      if (mode >= 1 && mode <= 7 && mode != 2) continue;
      if (mode == 7 && lg != 20) continue;
      float best = 1e30f, chk = 0.f;
      for (int rep = 0; rep < 4; ++rep) {
        CK(cudaMemset(out, 0, 4));
        cudaEventRecord(a);
        switch (mode) {
          case 0: k_ldgv<4, 0><<<nsm * 8, 256>>>(idx, E, tab, out); break;
          case 1: k_ldgv<8, 0><<<nsm * 8, 256>>>(idx, E, tab, out); break;
          case 2: k_ldgv<2, 0><<<nsm * 8, 256>>>(idx, E, tab, out); break;
          case 3: k_ldgv<1, 0><<<nsm * 8, 256>>>(idx, E, tab, out); break;
          case 4: k_ldgv<4, 1><<<nsm * 8, 256>>>(idx, E, tab, out); break;
          case 5: k_ldgv<2, 1><<<nsm * 8, 256>>>(idx, E, tab, out); break;
          case 6: k_ldg1<<<nsm * 8, 256>>>(idx, E, tab, out); break;
          case 8: k_rpl<8><<<nsm * 8, 256>>>(idx, E, tab, out); break;
          case 9: k_rpl<4><<<nsm * 8, 256>>>(idx, E, tab, out); break;
          case 10: k_rpl<2><<<nsm * 8, 256>>>(idx, E, tab, out); break;
          case 11: k_rpl<1><<<nsm * 8, 256>>>(idx, E, tab, out); break;
          case 7: k_tma<0><<<nsm, 32 * (NCW + 1), smem>>>(tm, idx, E, tab, out); break;
        }
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;
        CK(cudaMemcpy(&chk, out, 4, cudaMemcpyDeviceToHost));
      }
      printf("table %5.1f MB %-12s %7.3f ms  %6.1f Grows/s  %.2f cyc/row/SM  chk %.6e\n", rows * 64.0 / 1e6, nm[mode], best,
             E / best / 1e6, nsm * 1.965e9 / (E / best * 1e3), chk);
    }
  }
  return 0;
}
