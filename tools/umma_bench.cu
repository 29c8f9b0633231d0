// Microbenchmark: cost of one tcgen05.mma (kind::f16, bf16 in, fp32 accumulate)
// on B200 as a function of M, N, A-operand major-ness and A source (smem / TMEM),
// alone and with a concurrent 64 KB-per-tile bulk copy into shared memory (the
// K1 TMA stream). Answers: is the K1 MMA phase bound by the operand reads from
// shared memory (SS mode) rather than by the tensor MACs?
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/umma_bench tools/umma_bench.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2202_09512_b200/csrc/k1_tc.cuh"

using namespace rk::tc;

struct Mma {
  int n;       // N
  int m;       // M (64 or 128)
  int mn;      // A MN-major (1) or K-major (0)
  int ts;      // A from TMEM
};

struct Prog {
  int nmma;
  Mma mma[8];
};

__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "@px mov.s32 %0, 1;\n"
      "}\n"
      : "+r"(pred));
  return pred != 0;
}

// whole-warp issue: every lane runs the loop (warp-uniform descriptors in
// uniform registers), one elected lane executes the instruction
__device__ __forceinline__ void tc_mma_el(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, q;\n"
      "setp.ne.b32 q, %4, 0;\n"
      "elect.sync _|p, 0xffffffff;\n"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_el(uint32_t bar) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "elect.sync _|p, 0xffffffff;\n"
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(bar)
      : "memory");
}

// four MMAs behind one elect.sync (one asm block per k-step)
__device__ __forceinline__ void tc_mma4_el(uint32_t d0, uint64_t a0, uint64_t b0, uint32_t i0, uint32_t d1, uint64_t a1,
                                           uint64_t b1, uint32_t i1, uint32_t d2, uint64_t a2, uint64_t b2, uint32_t i2,
                                           uint32_t d3, uint64_t a3, uint64_t b3, uint32_t i3) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "elect.sync _|p, 0xffffffff;\n"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%4], %5, %6, %7, 1;\n"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%8], %9, %10, %11, 1;\n"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%12], %13, %14, %15, 1;\n"
      "}\n" ::"r"(d0),
      "l"(a0), "l"(b0), "r"(i0), "r"(d1), "l"(a1), "l"(b1), "r"(i1), "r"(d2), "l"(a2), "l"(b2), "r"(i2), "r"(d3),
      "l"(a3), "l"(b3), "r"(i3)
      : "memory");
}

__device__ __forceinline__ uint32_t idesc_m(int n, int m, int a_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// One MMA of the program: code = N | M << 10 | mn << 20 | ts << 21 (compile time,
// so the single issuing thread spends no time building descriptors).
template <int Code, bool EL>
__device__ __forceinline__ void issue_one(uint32_t d, uint32_t x, uint32_t bb, uint32_t tmem, int ks) {
  constexpr int N = Code & 1023, M = (Code >> 10) & 1023, MN = (Code >> 20) & 1, TS = (Code >> 21) & 1;
  constexpr uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)MN << 15) | ((uint32_t)(N >> 3) << 17) |
                          ((uint32_t)(M >> 4) << 24);
  const uint64_t db = umma_desc(bb + (ks & 3) * 32, 16, 1024);
  if (TS)
    tc_mma_ts(d, tmem + 448 + ks * 8, db, id, 1u);
  else if (EL && MN) {
    if (elect_one()) tc_mma(d, umma_desc(x + ks * 16 * 128, kXBox, 1024), db, id, 1u);
  } else if (EL) {
    if (elect_one()) tc_mma(d, umma_desc(x + (ks >> 2) * kXBox + (ks & 3) * 32, 16, 1024), db, id, 1u);
  }
  else if (MN)
    tc_mma(d, umma_desc(x + ks * 16 * 128, kXBox, 1024), db, id, 1u);
  else
    tc_mma(d, umma_desc(x + (ks >> 2) * kXBox + (ks & 3) * 32, 16, 1024), db, id, 1u);
}

template <bool EL, int... Codes>
__device__ __forceinline__ void issue_ks(uint32_t tmem, uint32_t dbase, uint32_t x, uint32_t bb, int ks) {
  // accumulator: bits 22..24 of the code (D = dbase + (acc & 3) * 64 columns)
  ((issue_one<Codes, EL>(dbase + (uint32_t)((Codes >> 22) & 3) * 64, x, bb, tmem, ks)), ...);
}

// mode bit0: run MMAs, bit1: run the copy stream. out[2*cta] = issuer cycles, out[2*cta+1] = copy cycles
template <int... Codes>
__global__ void __launch_bounds__(128, 1) bench(int tiles, int mode, const uint8_t* gsrc, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // layout: [0, 64K) operand X tile (hi+lo: 4 boxes of 16 KB), [64K, 96K) B operands,
  //         [96K, 160K) copy target, bars at 160K
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 160 * 1024);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 12);
  // warp index through a shuffle: provably warp-uniform for ptxas (uniform datapath)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 40 * 1024; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    mbar_init(smem_u32(&bars[1]), 1);
    for (int i = 2; i < 7; ++i) mbar_init(smem_u32(&bars[i]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0 && lane == 0) {
    unsigned long long t0 = clock64();
    if (mode & 2) {
      // 64 KB per tile into [96K, 160K) as 4 x 16 KB bulk copies (L2-resident source)
      uint32_t ph = 0;
      const uint8_t* src = gsrc + (size_t)(blockIdx.x & 63) * 65536;
      for (int t = 0; t < tiles; ++t) {
        const uint32_t b = smem_u32(&bars[0]);
        mbar_expect_tx(b, 65536);
        for (int q = 0; q < 4; ++q) bulk_g2s(smem_u32(smem + 96 * 1024 + q * 16384), src + q * 16384, 16384, b);
        mbar_wait(b, ph);
        ph ^= 1;
      }
    }
    out[2 * blockIdx.x + 1] = clock64() - t0;
  }
  const int nw = ((mode >> 2) & 3) + 1;  // issuing warps: 1..3 (warps 1..nw)
  if ((mode & 32) && warp == 1) {
    unsigned long long t0 = clock64();
    uint64_t* mb = bars + 1;
    const uint32_t x = smem_u32(smem), bb = smem_u32(smem + 64 * 1024);
    constexpr uint32_t i64k = (1u << 4) | (1u << 7) | (1u << 10) | (8u << 17) | (8u << 24);
    constexpr uint32_t i32k = (1u << 4) | (1u << 7) | (1u << 10) | (4u << 17) | (8u << 24);
    constexpr uint32_t i64m = i64k | (1u << 15), i32m = i32k | (1u << 15);
    int my = 0;
    for (int t = 0; t < tiles; ++t, ++my) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint64_t db = umma_desc(bb + (ks & 3) * 32, 16, 1024);
        const uint64_t dk = umma_desc(x + (ks >> 2) * kXBox + (ks & 3) * 32, 16, 1024);
        const uint64_t dm = umma_desc(x + ks * 16 * 128, kXBox, 1024);
        tc_mma4_el(tmem, dk, db, i64k, tmem, dk + 2048, db, i32k, tmem + 128, dm, db, i64m, tmem + 128, dm + 2048, db,
                   i32m);
      }
      if (elect_one()) tc_commit(smem_u32(&mb[my & 1]));
      __syncwarp();
      if (my > 0) mbar_wait(smem_u32(&mb[(my - 1) & 1]), (uint32_t)(((my - 1) >> 1) & 1));
    }
    if (my > 0) mbar_wait(smem_u32(&mb[(my - 1) & 1]), (uint32_t)(((my - 1) >> 1) & 1));
    if (lane == 0) out[2 * blockIdx.x] = clock64() - t0;
  } else if ((mode & 16) && warp >= 1 && warp <= nw) {
    // whole-warp issuer, elect.sync per instruction
    unsigned long long t0 = clock64();
    const int w = warp - 1;
    uint64_t* mb = bars + 1 + 2 * w;
    const uint32_t dbase = tmem + (uint32_t)w * 256;
    if (mode & 1) {
      const uint32_t x = smem_u32(smem), bb = smem_u32(smem + 64 * 1024);
      int my = 0;
      for (int t = w; t < tiles; t += nw, ++my) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) issue_ks<true, Codes...>(tmem, dbase, x, bb, ks);
        if (elect_one()) tc_commit(smem_u32(&mb[my & 1]));
        __syncwarp();
        if (my > 0) mbar_wait(smem_u32(&mb[(my - 1) & 1]), (uint32_t)(((my - 1) >> 1) & 1));
      }
      if (my > 0) mbar_wait(smem_u32(&mb[(my - 1) & 1]), (uint32_t)(((my - 1) >> 1) & 1));
    }
    if (w == 0 && lane == 0) out[2 * blockIdx.x] = clock64() - t0;
  } else if (!(mode & 16) && warp >= 1 && warp <= nw && lane == 0) {
    unsigned long long t0 = clock64();
    const int w = warp - 1;
    uint64_t* mb = bars + 1 + 2 * w;
    const uint32_t dbase = tmem + (uint32_t)w * 256;
    if (mode & 1) {
      const uint32_t x = smem_u32(smem), bb = smem_u32(smem + 64 * 1024);
      int my = 0;
      for (int t = w; t < tiles; t += nw, ++my) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) issue_ks<false, Codes...>(tmem, dbase, x, bb, ks);
        tc_commit(smem_u32(&mb[my & 1]));
        if (my > 0) mbar_wait(smem_u32(&mb[(my - 1) & 1]), (uint32_t)(((my - 1) >> 1) & 1));
      }
      if (my > 0) mbar_wait(smem_u32(&mb[(my - 1) & 1]), (uint32_t)(((my - 1) >> 1) & 1));
    }
    if (w == 0) out[2 * blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

constexpr int C(int n, int m, int mn, int ts, int acc = 0) { return n | (m << 10) | (mn << 20) | (ts << 21) | (acc << 22); }

template <int... Codes>
void run_case(const char* name, int tiles, const uint8_t* g, unsigned long long* d_out, int nsm, int nw = 1,
              int el = 0) {
  constexpr int nm = sizeof...(Codes);
  const size_t smem = 160 * 1024 + 1024 + 256;
  cudaFuncSetAttribute(bench<Codes...>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  std::vector<unsigned long long> h(2 * nsm);
  for (int mode0 = 1; mode0 <= 3; mode0 += 2) {
    const int mode = mode0 | ((nw - 1) << 2) | (el == 1 ? 16 : el == 2 ? 32 : 0);
    bench<Codes...><<<nsm, 128, smem>>>(4, mode, g, d_out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: %s\n", name, cudaGetErrorString(e));
      exit(1);
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    bench<Codes...><<<nsm, 128, smem>>>(tiles, mode, g, d_out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(h.data(), d_out, 2 * nsm * 8, cudaMemcpyDeviceToHost);
    unsigned long long mi = 0, mc = 0;
    for (int i = 0; i < nsm; ++i) {
      mi = h[2 * i] > mi ? h[2 * i] : mi;
      mc = h[2 * i + 1] > mc ? h[2 * i + 1] : mc;
    }
    const char* tag = mode0 == 1 ? "mma " : "both";
    printf("%-40s w%d%s %s  mma cyc/tile %7.1f (cyc/mma %6.1f)  copy cyc/tile %7.1f  %.3f ms  clk~%.0f MHz\n", name, nw, el == 2 ? "B" : el ? "E" : " ", tag,
           (double)mi / tiles, (double)mi / tiles / (8.0 * nm), (double)mc / tiles, ms,
           (double)(mi > mc ? mi : mc) / (ms * 1e3));
  }
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int nsm = 148;
  int tiles = argc > 1 ? atoi(argv[1]) : 2000;
  uint8_t* g;
  cudaMalloc(&g, 64 * 65536);
  cudaMemset(g, 0, 64 * 65536);
  unsigned long long* d_out;
  cudaMalloc(&d_out, 2 * nsm * sizeof(unsigned long long));
  printf("tiles=%d (8 k-steps each), grid=%d, 1 CTA/SM; copy = 64 KB bulk copy per tile\n", tiles, nsm);
  run_case<C(64, 128, 0, 0, 0), C(32, 128, 0, 0, 0), C(64, 128, 1, 0, 2), C(32, 128, 1, 0, 2)>(
      "mergedQ P(N64,N32) Q(N64,N32)", tiles, g, d_out, nsm, 1, 0);
  run_case<C(64, 128, 0, 0, 0), C(32, 128, 0, 0, 0), C(64, 128, 1, 0, 2), C(32, 128, 1, 0, 2)>(
      "mergedQ P(N64,N32) Q(N64,N32)", tiles, g, d_out, nsm, 1, 1);
  run_case<C(64, 128, 0, 0, 0), C(32, 128, 0, 0, 0), C(64, 128, 1, 0, 2), C(32, 128, 1, 0, 2)>(
      "mergedQ block-asm (4 MMAs / elect)", tiles, g, d_out, nsm, 1, 2);
  return 0;
}
