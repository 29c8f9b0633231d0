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

#include "k1_tc.cuh"
#include "rk_common.cuh"

namespace rk {
namespace sp {

RK_DEV uint32_t sp_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
RK_DEV void sp_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sp_smem_u32(dst)), "l"(src) : "memory");
}
RK_DEV void sp_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
RK_DEV void sp_cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

RK_DEV uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

RK_DEV void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

RK_DEV void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}


// L2 cache-policy helpers (createpolicy + .L2::cache_hint): the index/value
// streams and the output rows are touched once per pass (evict_first), the
// gathered factor rows are re-read ~10x per pass from L2 (evict_last, and not
// allocated in L1 where a random 64 B row is never reused).
RK_DEV uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
RK_DEV uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
RK_DEV int ld_stream(const int* a, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
RK_DEV float ld_stream(const float* a, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
  return v;
}
RK_DEV float4 ld_gather(const float* a, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(a), "l"(pol));
  return v;
}
RK_DEV void st_stream(float* a, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(a), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}

// SpMM pass Y_t = X_t B over the M slices of a CSR (or CSC) array set: one
// lane group of G = K/4 lanes per row, K accumulators as one float4 per lane,
// each stored entry gathers one K*4-byte row of B (coalesced across the group,
// L2-resident). Used for P_t = X_t A (CSR, rows) and Q_t = X_t^T A (CSC,
// columns). n = major dimension (rows of the block), Npad = row stride of Y.
// The (slice, row) task index advances incrementally (no 64-bit division per
// row); the gather loop keeps 4 independent loads in flight per lane; 32
// registers -> 64 resident warps per SM (the pass is L1/L2-latency bound).
template <int K>
#ifndef RK_SPC_MINB
#define RK_SPC_MINB 8
#endif
#ifndef RK_SPC_UNR
#define RK_SPC_UNR 4
#endif
__global__ void __launch_bounds__(256, RK_SPC_MINB) sp_csr_pass(const Ctl* __restrict__ ctl,
                                                      const int64_t* __restrict__ ptr,
                                                      const int* __restrict__ idx,
                                                      const float* __restrict__ val,
                                                      const float* __restrict__ A32,
                                                      float* __restrict__ P, int n, int Npad, int M,
                                                      int skip_if_stopped, int64_t a_stride = 0) {
  // a_stride > 0: slice t gathers from its own table A32 + t * a_stride (the
  // NNDSVD Gram products sum_t X_t B_t, rk_gram_apply)
  if (skip_if_stopped && ctl->stop) return;
  constexpr int G = K / 4;
  const uint64_t pf = l2_evict_first(), pl = l2_evict_last();
  const int lane = threadIdx.x & 31;
  const int q = lane % G;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int ngroups = (int)(((int64_t)gridDim.x * blockDim.x) / G);
  if (n <= 0) return;
  int t = (int)(group / n), i = (int)(group - (int64_t)t * n);
  for (; t < M;) {
    const int64_t* pt = ptr + (size_t)t * (n + 1);
    const int64_t b = pt[i], e = pt[i + 1];
    const float* At = A32 + (size_t)t * a_stride;
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t p = b;
    for (; p + RK_SPC_UNR <= e; p += RK_SPC_UNR) {
      int j[RK_SPC_UNR];
      float v[RK_SPC_UNR];
      float4 a[RK_SPC_UNR];
#pragma unroll
      for (int u = 0; u < RK_SPC_UNR; ++u) {
        j[u] = ld_stream(idx + p + u, pf);
        v[u] = ld_stream(val + p + u, pf);
      }
#pragma unroll
      for (int u = 0; u < RK_SPC_UNR; ++u) a[u] = ld_gather(At + (size_t)j[u] * K + 4 * q, pl);
#pragma unroll
      for (int u = 0; u < RK_SPC_UNR; ++u) {
        y.x = fmaf(v[u], a[u].x, y.x);
        y.y = fmaf(v[u], a[u].y, y.y);
        y.z = fmaf(v[u], a[u].z, y.z);
        y.w = fmaf(v[u], a[u].w, y.w);
      }
    }
    for (; p < e; ++p) {
      const int j = ld_stream(idx + p, pf);
      const float v = ld_stream(val + p, pf);
      const float4 a = ld_gather(At + (size_t)j * K + 4 * q, pl);
      y.x = fmaf(v, a.x, y.x);
      y.y = fmaf(v, a.y, y.y);
      y.z = fmaf(v, a.z, y.z);
      y.w = fmaf(v, a.w, y.w);
    }
    st_stream(P + ((size_t)t * Npad + i) * K + 4 * q, y, pf);
    i += ngroups;
    while (i >= n) {
      i -= n;
      ++t;
    }
  }
}

// S_t = A^T P_t (slots 1..M) and G = A^T A (slot 0) for tall P (sparse path,
// n up to 2^20+): a persistent grid walks (slot, row-chunk) items; each item
// streams its chunk's A and P_t rows through a 4-stage cp.async ring in shared
// memory; thread (c-block, d-block, row lane) forms a 4x4 block of the k x k
// outer-product sum in fp32 over <= 16 rows, then adds into fp64. The row
// lanes are summed in fixed order and each item writes one fp64 partial;
// sp_gram_reduce sums the chunk partials in chunk order (deterministic, no
// atomics). Replaces K2a (rk_kernels.cuh k2a_v4) on the sparse path, where
// the cluster-per-slot layout cannot stream 2 GB of P at HBM rate.
template <int K>
struct SpGramCfg {
  static constexpr int KB = K / 4;
  static constexpr int NB = KB * KB;     // 4x4 blocks
  static constexpr int RL = 256 / NB;    // row lanes
  static constexpr int SR = K == 16 ? 128 : 64;  // rows per stage
  static constexpr int RPT = SR / RL;            // rows per thread per stage (8 | 16)
  static constexpr int NS = 6;           // stages (2 CTAs/SM: ~160 KB in flight)
  static constexpr size_t smem = (size_t)NS * SR * K * 2 * sizeof(float);
};

template <int K>
__global__ void __launch_bounds__(256) sp_gram(const Ctl* __restrict__ ctl, const float* __restrict__ A32,
                                               const float* __restrict__ P, int n, int ldp, int M,
                                               int nchunk, double* __restrict__ part,
                                               int skip_if_stopped) {
  using C = SpGramCfg<K>;
  if (skip_if_stopped && ctl->stop) return;
  extern __shared__ __align__(16) float gsm[];
  float* As = gsm;
  float* Bs = gsm + C::NS * C::SR * K;
  const int tid = threadIdx.x;
  const int sub = tid % C::NB, rl = tid / C::NB;
  const int cb = sub / C::KB, db = sub % C::KB;
  const int rows_per_chunk = (n + nchunk - 1) / nchunk;
  const int nitems = (M + 1) * nchunk;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int slot = item / nchunk, chunk = item - slot * nchunk;
    const float* B = slot == 0 ? A32 : P + (size_t)(slot - 1) * ldp * K;
    const int r0 = chunk * rows_per_chunk, r1 = min(n, r0 + rows_per_chunk);
    const int nst = r1 > r0 ? (r1 - r0 + C::SR - 1) / C::SR : 0;
    auto issue = [&](int s) {
      const int base = r0 + s * C::SR, nr = min(C::SR, r1 - base);
      float* as = As + (s % C::NS) * C::SR * K;
      float* bs = Bs + (s % C::NS) * C::SR * K;
      for (int e = tid; e < nr * (K / 4); e += 256) {
        sp_cp16(as + 4 * e, A32 + (size_t)base * K + 4 * e);
        sp_cp16(bs + 4 * e, B + (size_t)base * K + 4 * e);
      }
    };
    __syncthreads();  // previous item's buffers fully consumed
#pragma unroll
    for (int s = 0; s < C::NS - 1; ++s) {
      if (s < nst) issue(s);
      sp_cp_commit();
    }
    double acc[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) acc[u] = 0.0;
    float pacc[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) pacc[u] = 0.f;
    for (int s = 0; s < nst; ++s) {
      if (s + C::NS - 1 < nst) issue(s + C::NS - 1);
      sp_cp_commit();
      sp_cp_wait<C::NS - 1>();
      __syncthreads();
      const int nr = min(C::SR, r1 - (r0 + s * C::SR));
      const float* as = As + (s % C::NS) * C::SR * K;
      const float* bs = Bs + (s % C::NS) * C::SR * K;
      auto row = [&](int r) {
        const float4 a = *reinterpret_cast<const float4*>(as + r * K + 4 * cb);
        const float4 b = *reinterpret_cast<const float4*>(bs + r * K + 4 * db);
        const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) pacc[x * 4 + y] = fmaf(av[x], bv[y], pacc[x * 4 + y]);
      };
      if (nr == C::SR) {
#pragma unroll
        for (int u = 0; u < C::RPT; ++u) row(rl + u * C::RL);
      } else {
        for (int r = rl; r < nr; r += C::RL) row(r);
      }
      // fp32 chains of <= 16 rows, then fp64
      if (C::RPT >= 16 || (s & 1) || s == nst - 1) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          acc[u] += (double)pacc[u];
          pacc[u] = 0.f;
        }
      }
      __syncthreads();  // buffer s % NS is refilled by the next iteration
    }
    // row-lane reduction in fixed order through shared memory (reuses the ring)
    double* red = reinterpret_cast<double*>(gsm);
    sp_cp_wait<0>();
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) red[(size_t)rl * (C::NB * 16) + sub * 16 + u] = acc[u];
    __syncthreads();
    for (int o = tid; o < K * K; o += 256) {
      double v = 0.0;
      for (int l = 0; l < C::RL; ++l) v += red[(size_t)l * (C::NB * 16) + o];
      const int sb = o / 16, u = o % 16;
      const int c = (sb / C::KB) * 4 + u / 4, d = (sb % C::KB) * 4 + u % 4;
      part[((size_t)slot * nchunk + chunk) * K * K + c * K + d] = v;
    }
  }
}

// Tensor-core form of sp_gram for K = 16: S = A^T B over a row chunk is an
// m16n8k8 TF32 product with the rows as the K dimension (3-pass split,
// truncation hi / exact lo as in sp_numer_tc). Index permutations make every
// fragment an LDS.64: output row m <-> c = 2g (m = g) / 2g+1 (m = g+8), output
// column n of n-tile nt <-> d = 2n + nt, so lane (g, tq) reads columns 2g, 2g+1
// of rows tq and tq+4 of the 8-row k-step from both A and B; rows are padded
// to 24 floats (conflict-free). fp32 accumulation over <= 32 rows per warp,
// then fp64; warp partials summed in fixed order; one fp64 partial per item.
#ifndef RK_SG_NS
#define RK_SG_NS 2
#endif
#ifndef RK_SG_CPS
#define RK_SG_CPS 4
#endif
struct SpGramTc {
  static constexpr int K = 16, SR = 128, LD = 24, NS = RK_SG_NS;
  static constexpr int CPS = RK_SG_CPS;  // CTAs per SM
  static constexpr int ARR = SR * LD;  // floats per array per stage
  static constexpr size_t smem = (size_t)NS * 2 * ARR * sizeof(float);  // 48 KB (>= 8 warps x 256 doubles)
};

// KT = 32 / 48 / 64 (dense): each (slot, chunk) item is split into the
// (KT/16)^2 16 x 16 column blocks of S (item-minor), each the K = 16 product
// above on column slices of the KT-wide rows; blocks write disjoint partial
// entries.
// Body over the items bid, bid + nblk, ... (also phase 2 of the fused
// k-wide chain, k2_chain.cuh); gts: the block's >= SpGramTc::smem bytes.
template <int KT>
RK_DEV void sp_gram_tc_body(const float* __restrict__ A32, const float* __restrict__ P, int n, int ldp, int M,
                            int nchunk, double* __restrict__ part, const float* __restrict__ Aown, int nown,
                            int bid, int nblk, float* gts) {
  // slot 0 (G) runs over Aown's nown rows when given (a grid rank's own piece
  // of A, rescal.py:124 with the grid's rank-ascending sum, dist_rescal.py:74-92)
  using C = SpGramTc;
  static_assert(KT == 16 || KT == 32 || KT == 48 || KT == 64, "sp_gram_tc_k: K in {16, 32, 48, 64}");
  constexpr int NQ1 = KT / 16, NQ = NQ1 * NQ1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int rows_per_chunk = (n + nchunk - 1) / nchunk;
  // a block takes whole (slot, chunk) groups (all NQ quadrant items of the
  // same rows): the fused chain reduces exactly those P rows just before
  const int nitems = (M + 1) * nchunk * NQ;
  for (int item0 = bid * NQ; item0 < nitems; item0 += nblk * NQ)
  for (int item = item0; item < item0 + NQ; ++item) {
    const int q = item % NQ, sc = item / NQ;
    const int slot = sc / nchunk, chunk = sc - slot * nchunk;
    const int ca = (q / NQ1) * 16, cb = (q % NQ1) * 16;
    const bool own = slot == 0 && Aown != nullptr;
    const float* Ai = own ? Aown : A32;
    const float* B = slot == 0 ? Ai : P + (size_t)(slot - 1) * ldp * KT;
    const int nn = own ? nown : n;
    const int rpc = own ? (nown + nchunk - 1) / nchunk : rows_per_chunk;
    const int r0 = chunk * rpc, r1 = min(nn, r0 + rpc);
    const int nst = r1 > r0 ? (r1 - r0 + C::SR - 1) / C::SR : 0;
    auto issue = [&](int s) {
      const int base = r0 + s * C::SR, nr = min(C::SR, r1 - base);
      float* as = gts + (size_t)(s % C::NS) * 2 * C::ARR;
      float* bs = as + C::ARR;
      for (int e = tid; e < C::SR * 4; e += 256) {
        const int r = e >> 2, c4 = e & 3;
        if (r < nr) {
          sp_cp16(as + r * C::LD + 4 * c4, Ai + (size_t)(base + r) * KT + ca + 4 * c4);
          sp_cp16(bs + r * C::LD + 4 * c4, B + (size_t)(base + r) * KT + cb + 4 * c4);
        } else {  // rows past the chunk contribute zero
          *reinterpret_cast<float4*>(as + r * C::LD + 4 * c4) = make_float4(0.f, 0.f, 0.f, 0.f);
          *reinterpret_cast<float4*>(bs + r * C::LD + 4 * c4) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    };
    __syncthreads();  // previous item's buffers (and reduction scratch) consumed
#pragma unroll
    for (int s = 0; s < C::NS - 1; ++s) {
      if (s < nst) issue(s);
      sp_cp_commit();
    }
    double acc[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int x = 0; x < 4; ++x) acc[nt][x] = 0.0;
    float c[2][4];
    for (int s = 0; s < nst; ++s) {
      if (s + C::NS - 1 < nst) issue(s + C::NS - 1);
      sp_cp_commit();
      sp_cp_wait<C::NS - 1>();
      __syncthreads();
      const float* as = gts + (size_t)(s % C::NS) * 2 * C::ARR;
      const float* bs = as + C::ARR;
      if ((s & 1) == 0) {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int x = 0; x < 4; ++x) c[nt][x] = 0.f;
      }
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {  // this warp's two 8-row k-steps of the stage
        const int rb = (warp + 8 * kk) * 8;
        const float2 a_lo_row = *reinterpret_cast<const float2*>(as + (rb + tq) * C::LD + 2 * g);
        const float2 a_hi_row = *reinterpret_cast<const float2*>(as + (rb + tq + 4) * C::LD + 2 * g);
        const float2 b_lo_row = *reinterpret_cast<const float2*>(bs + (rb + tq) * C::LD + 2 * g);
        const float2 b_hi_row = *reinterpret_cast<const float2*>(bs + (rb + tq + 4) * C::LD + 2 * g);
        const float av[4] = {a_lo_row.x, a_lo_row.y, a_hi_row.x, a_hi_row.y};
        uint32_t ah[4], al[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          ah[q] = __float_as_uint(av[q]) & 0xffffe000u;
          al[q] = __float_as_uint(av[q] - __uint_as_float(ah[q]));
        }
        // n-tile nt: b0 = B[row tq][2g + nt], b1 = B[row tq+4][2g + nt]
        const float bv[2][2] = {{b_lo_row.x, b_hi_row.x}, {b_lo_row.y, b_hi_row.y}};
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const uint32_t bh0 = __float_as_uint(bv[nt][0]) & 0xffffe000u, bh1 = __float_as_uint(bv[nt][1]) & 0xffffe000u;
          const uint32_t bl0 = __float_as_uint(bv[nt][0] - __uint_as_float(bh0));
          const uint32_t bl1 = __float_as_uint(bv[nt][1] - __uint_as_float(bh1));
          mma_tf32(c[nt], al, bh0, bh1);
          mma_tf32(c[nt], ah, bl0, bl1);
          mma_tf32(c[nt], ah, bh0, bh1);
        }
      }
      if ((s & 1) || s == nst - 1) {  // fp32 over <= 32 rows per lane product, then fp64
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int x = 0; x < 4; ++x) acc[nt][x] += (double)c[nt][x];
      }
      __syncthreads();  // buffer s % NS is refilled by the next iteration
    }
    // warp partials -> fixed-order sum; lane (g, tq) holds
    // c_nt[0] = S[2g][4tq+nt], c_nt[1] = S[2g][4tq+2+nt], c_nt[2] = S[2g+1][4tq+nt], c_nt[3] = S[2g+1][4tq+2+nt]
    sp_cp_wait<0>();
    __syncthreads();
    double* red = reinterpret_cast<double*>(gts);  // [8 warps][256]
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      red[warp * 256 + (2 * g) * 16 + 4 * tq + nt] = acc[nt][0];
      red[warp * 256 + (2 * g) * 16 + 4 * tq + 2 + nt] = acc[nt][1];
      red[warp * 256 + (2 * g + 1) * 16 + 4 * tq + nt] = acc[nt][2];
      red[warp * 256 + (2 * g + 1) * 16 + 4 * tq + 2 + nt] = acc[nt][3];
    }
    __syncthreads();
    {
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) v += red[w * 256 + tid];
      part[((size_t)slot * nchunk + chunk) * KT * KT + (ca + (tid >> 4)) * KT + cb + (tid & 15)] = v;
    }
  }
}

template <int KT>
__global__ void __launch_bounds__(256, RK_SG_CPS) sp_gram_tc_k(const Ctl* __restrict__ ctl, const float* __restrict__ A32,
                                                     const float* __restrict__ P, int n, int ldp, int M, int nchunk,
                                                     double* __restrict__ part, int skip_if_stopped,
                                                     const float* __restrict__ Aown = nullptr, int nown = 0) {
  if (skip_if_stopped && ctl->stop) return;
  extern __shared__ __align__(16) float gts[];
  sp_gram_tc_body<KT>(A32, P, n, ldp, M, nchunk, part, Aown, nown, blockIdx.x, gridDim.x, gts);
}

__global__ void __launch_bounds__(256) sp_gram_reduce(const Ctl* __restrict__ ctl,
                                                      const double* __restrict__ part, int nchunk,
                                                      int KK, double* __restrict__ gs,
                                                      int skip_if_stopped) {
  if (skip_if_stopped && ctl->stop) return;
  const int slot = blockIdx.x;
  for (int e = threadIdx.x; e < KK; e += blockDim.x)
    gs[(size_t)slot * KK + e] = sum_chunks(part + (size_t)slot * nchunk * KK + e, nchunk, KK);
}

// A update from the stored P_t = X_t A and Q_t = X_t^T A (sparse path):
//   num_i = sum_t P_t[i] R_t^T + Q_t[i] R_t      (rescal.py:133-143)
//   A_i <- A_i * num_i / (A_i M + m eps)         (rescal.py:144-145)
// Persistent: one CTA per SM walks its row blocks; the flat sequence of
// (row block, slice t) stages — the block's P_t / Q_t rows plus W_t =
// [R_t^T ; R_t] (fp32, written by the K2f commit) — streams through a
// cp.async ring in shared memory without draining between row blocks (P/Q
// row stride padded to K+4 floats: conflict-free LDS.128). Thread = NRT rows
// x 4 output columns; per slice the 2K-term products are formed in fp32 and
// accumulated across slices in fp64 (as k2b_v4). A row block's update is
// applied after its last slice; each CTA owns its rows, so the in-place A
// update is race-free.
template <int K>
struct SpNumCfg {
  static constexpr int NRT = 2;         // rows per thread
  static constexpr int CB = K / 4;
  static constexpr int RQ = 256 / CB;   // row lanes
  static constexpr int RB = NRT * RQ;   // rows per block
  static constexpr int LD = K + 4;      // padded smem row (floats)
  static constexpr int NS = 4;          // ring stages
  static constexpr int STAGE = 2 * RB * LD + 2 * K * K;  // floats per stage
  static constexpr size_t smem = (size_t)NS * STAGE * sizeof(float) + (size_t)K * K * sizeof(double);
};

template <int K>
__global__ void __launch_bounds__(256, 2) sp_numer_apply(Ctl* __restrict__ ctl, double* __restrict__ A64,
                                                         float* __restrict__ A32,
                                                         const float* __restrict__ P,
                                                         const float* __restrict__ Q, int ldp, int ldq,
                                                         const float* __restrict__ W32,
                                                         const double* __restrict__ Mm, int n, int M,
                                                         double eps_m) {
  using C = SpNumCfg<K>;
  if (ctl->stop) return;
  extern __shared__ __align__(16) float nsm[];
  double* Ms = reinterpret_cast<double*>(nsm + (size_t)C::NS * C::STAGE);
  const int tid = threadIdx.x;
  const int cb = tid % C::CB, rq = tid / C::CB;
  const int nrb = (n + C::RB - 1) / C::RB;
  const int my_rb = nrb > (int)blockIdx.x ? (nrb - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int nstage = my_rb * M;
  if (nstage == 0) return;
  for (int e = tid; e < K * K; e += 256) Ms[e] = Mm[e];
  auto issue = [&](int f) {
    const int t = f % M, row0 = ((int)blockIdx.x + (f / M) * (int)gridDim.x) * C::RB;
    const int nr = min(C::RB, n - row0);
    float* ps = nsm + (size_t)(f % C::NS) * C::STAGE;
    float* qs = ps + C::RB * C::LD;
    float* ws = qs + C::RB * C::LD;
    const float* pg = P + ((size_t)t * ldp + row0) * K;
    const float* qg = Q + ((size_t)t * ldq + row0) * K;
    for (int e = tid; e < nr * (K / 4); e += 256) {
      const int r = e / (K / 4), c4 = e % (K / 4);
      sp_cp16(ps + r * C::LD + 4 * c4, pg + (size_t)r * K + 4 * c4);
      sp_cp16(qs + r * C::LD + 4 * c4, qg + (size_t)r * K + 4 * c4);
    }
    for (int e = tid; e < 2 * K * K / 4; e += 256) sp_cp16(ws + 4 * e, W32 + (size_t)t * 2 * K * K + 4 * e);
  };
#pragma unroll
  for (int s = 0; s < C::NS - 1; ++s) {
    if (s < nstage) issue(s);
    sp_cp_commit();
  }
  double acc[C::NRT][4];
  bool bad = false;
  for (int f = 0; f < nstage; ++f) {
    const int t = f % M;
    const int row0 = ((int)blockIdx.x + (f / M) * (int)gridDim.x) * C::RB;
    const int nr = min(C::RB, n - row0);
    if (f + C::NS - 1 < nstage) issue(f + C::NS - 1);
    sp_cp_commit();
    sp_cp_wait<C::NS - 1>();
    __syncthreads();
    if (t == 0) {
#pragma unroll
      for (int u = 0; u < C::NRT; ++u)
#pragma unroll
        for (int x = 0; x < 4; ++x) acc[u][x] = 0.0;
    }
    const float* ps = nsm + (size_t)(f % C::NS) * C::STAGE;
    const float* qs = ps + C::RB * C::LD;
    const float* WrT = qs + C::RB * C::LD;  // [d][c] = R_t[c][d]
    const float* Wr = WrT + K * K;          // [d][c] = R_t[d][c]
    float s[C::NRT][4];
#pragma unroll
    for (int u = 0; u < C::NRT; ++u)
#pragma unroll
      for (int x = 0; x < 4; ++x) s[u][x] = 0.f;
#pragma unroll
    for (int d4 = 0; d4 < K / 4; ++d4) {
      float4 pr[C::NRT], qr[C::NRT];
#pragma unroll
      for (int u = 0; u < C::NRT; ++u) {
        const int r = rq + u * C::RQ;
        pr[u] = *reinterpret_cast<const float4*>(ps + r * C::LD + 4 * d4);
        qr[u] = *reinterpret_cast<const float4*>(qs + r * C::LD + 4 * d4);
      }
#pragma unroll
      for (int dd = 0; dd < 4; ++dd) {
        const int d = 4 * d4 + dd;
        const float4 wp = *reinterpret_cast<const float4*>(WrT + d * K + 4 * cb);
        const float4 wq = *reinterpret_cast<const float4*>(Wr + d * K + 4 * cb);
#pragma unroll
        for (int u = 0; u < C::NRT; ++u) {
          const float pv = dd == 0 ? pr[u].x : dd == 1 ? pr[u].y : dd == 2 ? pr[u].z : pr[u].w;
          const float qv = dd == 0 ? qr[u].x : dd == 1 ? qr[u].y : dd == 2 ? qr[u].z : qr[u].w;
          s[u][0] = fmaf(pv, wp.x, fmaf(qv, wq.x, s[u][0]));
          s[u][1] = fmaf(pv, wp.y, fmaf(qv, wq.y, s[u][1]));
          s[u][2] = fmaf(pv, wp.z, fmaf(qv, wq.z, s[u][2]));
          s[u][3] = fmaf(pv, wp.w, fmaf(qv, wq.w, s[u][3]));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < C::NRT; ++u)
#pragma unroll
      for (int x = 0; x < 4; ++x) acc[u][x] += (double)s[u][x];
    if (t == M - 1) {
      // A update of this row block: read the old rows, sync, write
      double an[C::NRT][4];
#pragma unroll
      for (int u = 0; u < C::NRT; ++u) {
        const int r = rq + u * C::RQ;
        if (r < nr) {
          const double* Ai = A64 + (size_t)(row0 + r) * K;
          double deno[4] = {eps_m, eps_m, eps_m, eps_m};
          for (int d = 0; d < K; ++d) {
            const double a = Ai[d];
#pragma unroll
            for (int x = 0; x < 4; ++x) deno[x] = fma(a, Ms[d * K + 4 * cb + x], deno[x]);
          }
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            an[u][x] = Ai[4 * cb + x] * acc[u][x] / deno[x];
            bad |= !isfinite(an[u][x]);
          }
        }
      }
      __syncthreads();  // every thread has read its whole A rows before any write
#pragma unroll
      for (int u = 0; u < C::NRT; ++u) {
        const int r = rq + u * C::RQ;
        if (r < nr) {
          double* Ai = A64 + (size_t)(row0 + r) * K + 4 * cb;
          float* Af = A32 + (size_t)(row0 + r) * K + 4 * cb;
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            Ai[x] = an[u][x];
            Af[x] = (float)an[u][x];
          }
        }
      }
    }
    __syncthreads();  // stage f % NS is refilled next iteration
  }
  if (bad) {
    ctl->nonfinite = 1;
    ctl->stop = 1;
  }
}

// ---- tensor-core numerator (K = 16): num = [P_1..P_m Q_1..Q_m] . [R_t^T ; R_t]
// is an (n x 32m) by (32m x 16) GEMM. mma.sync m16n8k8 TF32 with the 3-pass
// split (a_hi b_hi + a_hi b_lo + a_lo b_hi, fp32-level products); a warp owns
// 32 rows (two m-tiles) x 16 columns. The K order inside a slice is permuted so
// that each lane's A fragment is one LDS.128 of a contiguous smem row (lane
// (g, tq) holds d = 4tq..4tq+3 of rows g and g+8: k-step s uses d = 4tq+2s and
// 4tq+2s+1), which is conflict-free on unpadded 64-byte rows. The matching B
// fragments (hi/lo, per slice) are laid out per lane by sp_wfrag.
// Wf[t][pq][s][nt][lane] = {b0_hi, b1_hi, b0_lo, b1_lo} with lane = 4g + tq,
// b0 = W[4tq+2s][8nt+g], b1 = W[4tq+2s+1][8nt+g], W = R_t^T (pq 0) | R_t (pq 1)
// taken from W32 = [R_t^T ; R_t] (K = 16).
__global__ void __launch_bounds__(256) sp_wfrag(const Ctl* __restrict__ ctl, const float* __restrict__ W32,
                                                float4* __restrict__ Wf, int M) {
  if (ctl->stop) return;
  const int t = blockIdx.x;
  const int lane = threadIdx.x & 31, combo = threadIdx.x >> 5;  // combo = pq*4 + s*2 + nt
  const int pq = combo >> 2, s = (combo >> 1) & 1, nt = combo & 1;
  const int g = lane >> 2, tq = lane & 3;
  const float* W = W32 + ((size_t)t * 2 + pq) * 256;
  const float b0 = W[(4 * tq + 2 * s) * 16 + 8 * nt + g], b1 = W[(4 * tq + 2 * s + 1) * 16 + 8 * nt + g];
  const uint32_t h0 = tf32_rna(b0), h1 = tf32_rna(b1);
  const uint32_t l0 = tf32_rna(b0 - __uint_as_float(h0)), l1 = tf32_rna(b1 - __uint_as_float(h1));
  Wf[((size_t)t * 8 + combo) * 32 + lane] =
      make_float4(__uint_as_float(h0), __uint_as_float(h1), __uint_as_float(l0), __uint_as_float(l1));
}

struct SpNumTc {
  static constexpr int K = 16;
  static constexpr int RB = 256;  // rows per row block (8 warps x 32)
  static constexpr int NS = 3;    // two CTAs per SM: ~140 KB in flight per SM
  static constexpr int PQ_BYTES = RB * K * 4;         // one of P_t / Q_t
  static constexpr int WF_BYTES = 8 * 32 * 16;        // Wf_t
  static constexpr int STAGE = 2 * PQ_BYTES + WF_BYTES;
  static constexpr size_t smem = (size_t)NS * STAGE + K * K * sizeof(double) + NS * 8 + 128;
};

__global__ void __launch_bounds__(256, 2) sp_numer_tc(Ctl* __restrict__ ctl, double* __restrict__ A64,
                                                      float* __restrict__ A32, const float* __restrict__ P,
                                                      const float* __restrict__ Q, int ldp, int ldq,
                                                      const float4* __restrict__ Wf,
                                                      const double* __restrict__ Mm, int n, int M,
                                                      double eps_m, int only = -1,
                                                      double* __restrict__ U = nullptr) {
  // only < 0: num from P and Q, then the A update (single GPU).
  // only = 0 | 1: U = sum_t Y_t R_t^T (0, Y = P) or sum_t Y_t R_t (1, Y passed
  // as P) written as fp64 rows — the grid's row / column numerator partials
  // before their reduce-scatter.
  using C = SpNumTc;
  constexpr int K = 16;
  if (ctl->stop) return;
  extern __shared__ __align__(128) uint8_t tsm[];
  uint8_t* ring = tsm;
  double* Ms = reinterpret_cast<double*>(tsm + (size_t)C::NS * C::STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(Ms + K * K);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int nrb = (n + C::RB - 1) / C::RB;
  const int my_rb = nrb > (int)blockIdx.x ? (nrb - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int nstage = my_rb * M;
  if (nstage == 0) return;
  for (int e = tid; e < K * K; e += 256) Ms[e] = Mm[e];
  if (tid == 0) {
    for (int i = 0; i < C::NS; ++i) tc::mbar_init(tc::smem_u32(&full[i]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int f) {  // thread 0 only
    const int t = f % M, row0 = ((int)blockIdx.x + (f / M) * (int)gridDim.x) * C::RB;
    const int nr = min(C::RB, n - row0);
    uint8_t* st = ring + (size_t)(f % C::NS) * C::STAGE;
    const uint32_t bar = tc::smem_u32(&full[f % C::NS]);
    const uint32_t bytes = (uint32_t)nr * K * 4;
    tc::mbar_expect_tx(bar, (only < 0 ? 2 : 1) * bytes + C::WF_BYTES);
    bulk_g2s(tc::smem_u32(st + (only > 0 ? C::PQ_BYTES : 0)), P + ((size_t)t * ldp + row0) * K, bytes, bar);
    if (only < 0) bulk_g2s(tc::smem_u32(st + C::PQ_BYTES), Q + ((size_t)t * ldq + row0) * K, bytes, bar);
    bulk_g2s(tc::smem_u32(st + 2 * C::PQ_BYTES), Wf + (size_t)t * 256, C::WF_BYTES, bar);
  };
  if (tid == 0)
    for (int f = 0; f < C::NS - 1 && f < nstage; ++f) issue(f);
  double acc[2][2][4];
  float c[2][2][4];  // [mt][nt][frag]
  bool bad = false;
  for (int f = 0; f < nstage; ++f) {
    const int t = f % M;
    const int row0 = ((int)blockIdx.x + (f / M) * (int)gridDim.x) * C::RB;
    const int nr = min(C::RB, n - row0);
    if (tid == 0 && f + C::NS - 1 < nstage) issue(f + C::NS - 1);
    tc::mbar_wait(tc::smem_u32(&full[f % C::NS]), (uint32_t)((f / C::NS) & 1));
    if (t == 0) {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int x = 0; x < 4; ++x) acc[mt][nt][x] = 0.0;
    }
    const uint8_t* st = ring + (size_t)(f % C::NS) * C::STAGE;
    const float4* wf = reinterpret_cast<const float4*>(st + 2 * C::PQ_BYTES);
    if ((t & 1) == 0) {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int x = 0; x < 4; ++x) c[mt][nt][x] = 0.f;
    }
#pragma unroll
    for (int pq = 0; pq < 2; ++pq) {
      if (only >= 0 && pq != only) continue;
      const float* S = reinterpret_cast<const float*>(st + pq * C::PQ_BYTES);
      float4 bw[2][2];
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) bw[s][nt] = wf[(pq * 4 + s * 2 + nt) * 32 + lane];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int r = warp * 32 + mt * 16 + g;
        const float4 x0 = *reinterpret_cast<const float4*>(S + r * K + 4 * tq);
        const float4 x1 = *reinterpret_cast<const float4*>(S + (r + 8) * K + 4 * tq);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const float v[4] = {s ? x0.z : x0.x, s ? x1.z : x1.x, s ? x0.w : x0.y, s ? x1.w : x1.y};
          uint32_t ah[4], al[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {  // hi = truncation to tf32 (one LOP), lo exact
            ah[q] = __float_as_uint(v[q]) & 0xffffe000u;
            al[q] = __float_as_uint(v[q] - __uint_as_float(ah[q]));
          }
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const float4 b = bw[s][nt];
            mma_tf32(c[mt][nt], al, __float_as_uint(b.x), __float_as_uint(b.y));
            mma_tf32(c[mt][nt], ah, __float_as_uint(b.z), __float_as_uint(b.w));
            mma_tf32(c[mt][nt], ah, __float_as_uint(b.x), __float_as_uint(b.y));
          }
        }
      }
    }
    if ((t & 1) || t == M - 1) {  // fp32 over <= 2 slices (64 products), then fp64
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int x = 0; x < 4; ++x) acc[mt][nt][x] += (double)c[mt][nt][x];
    }
    if (t == M - 1 && only >= 0) {
      // numerator partial rows (fp64): lane (g, tq) holds rows r / r + 8 at
      // columns 8nt + 2tq + {0, 1} of each m-tile
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = warp * 32 + mt * 16 + g + 8 * h;
          if (r < nr) {
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
              *reinterpret_cast<double2*>(U + (size_t)(row0 + r) * K + 8 * nt + 2 * tq) =
                  make_double2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]);
          }
        }
    } else if (t == M - 1) {
      // A update of this row block. Lane (g, tq) holds rows r (c0, c1) and
      // r + 8 (c2, c3) at columns 8nt + 2tq + {0, 1} of each m-tile. A row is
      // read and written only by the four lanes of one quad (same warp), so a
      // warp barrier orders each row's reads before its writes.
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = warp * 32 + mt * 16 + g + 8 * h;
          const bool ok = r < nr;
          double* Ai = A64 + (size_t)(row0 + (ok ? r : 0)) * K;
          double out[2][2];
          if (ok) {
            double deno[2][2] = {{eps_m, eps_m}, {eps_m, eps_m}};
#pragma unroll 4
            for (int d = 0; d < K; ++d) {
              const double a = Ai[d];
              const double2 m0 = *reinterpret_cast<const double2*>(Ms + d * K + 2 * tq);
              const double2 m1 = *reinterpret_cast<const double2*>(Ms + d * K + 8 + 2 * tq);
              deno[0][0] = fma(a, m0.x, deno[0][0]);
              deno[0][1] = fma(a, m0.y, deno[0][1]);
              deno[1][0] = fma(a, m1.x, deno[1][0]);
              deno[1][1] = fma(a, m1.y, deno[1][1]);
            }
            const double2 a0 = *reinterpret_cast<const double2*>(Ai + 2 * tq);
            const double2 a1 = *reinterpret_cast<const double2*>(Ai + 8 + 2 * tq);
            out[0][0] = a0.x * acc[mt][0][2 * h] / deno[0][0];
            out[0][1] = a0.y * acc[mt][0][2 * h + 1] / deno[0][1];
            out[1][0] = a1.x * acc[mt][1][2 * h] / deno[1][0];
            out[1][1] = a1.y * acc[mt][1][2 * h + 1] / deno[1][1];
            bad |= !(isfinite(out[0][0]) && isfinite(out[0][1]) && isfinite(out[1][0]) && isfinite(out[1][1]));
          }
          __syncwarp();
          if (ok) {
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              const int col = 8 * nt + 2 * tq;
              *reinterpret_cast<double2*>(Ai + col) = make_double2(out[nt][0], out[nt][1]);
              *reinterpret_cast<float2*>(A32 + (size_t)(row0 + r) * K + col) =
                  make_float2((float)out[nt][0], (float)out[nt][1]);
            }
          }
          __syncwarp();
        }
    }
    __syncthreads();  // stage f % NS is refilled next iteration
  }
  if (bad) {
    ctl->nonfinite = 1;
    ctl->stop = 1;
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
      const double f = pcg_field(u, delta);
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

// Upload helpers (host CSR -> device, validated on the device): rebase a
// slice's local indptr to global offsets; check column ids; check values
// (non-negative, tensor.py:102-103), convert to fp32 and form per-block fp64
// sums of squares (||X||^2, rescal.py:160-165) in a fixed order.
__global__ void sp_rebase_ptr(const int64_t* __restrict__ src, int64_t count, int64_t base,
                              int64_t* __restrict__ dst) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = src[e] + base;
}

__global__ void sp_check_idx(const int* __restrict__ idx, int64_t count, int cols, int* __restrict__ flag) {
  bool bad = false;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int j = idx[e];
    bad |= j < 0 || j >= cols;
  }
  if (bad) atomicOr(flag, 2);
}

template <typename T>
__global__ void __launch_bounds__(256) sp_take_vals(const T* __restrict__ src, int64_t count,
                                                    float* __restrict__ dst, double* __restrict__ part,
                                                    int* __restrict__ flag) {
  __shared__ double red[8];
  double acc = 0.0;
  bool bad = false;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)src[e];
    bad |= !(v >= 0.0);
    acc += v * v;
    dst[e] = (float)v;
  }
  if (bad) atomicOr(flag, 1);
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
