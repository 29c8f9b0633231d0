// EXPERIMENT (not built into librescal_b200.so). Round 2 wired this kernel in
// place of k2b_v4 for the dense one-GPU A update (fragments written by k2f):
// cfg3 k2b 166 -> 69 us (ncu), but k2f grew by the fragment writes, the
// persistent grid under-fills small problems (cfg1 34.7k -> 29.5k it/s), cfg2
// and cfg3 were unchanged within the box-to-box clock noise, and the cfg1
// 200-iteration parity test against the reference golden moved from relR
// ~1e-5 to 1.13e-4 (> the 1e-4 tolerance): the TF32 3-pass products and the
// tensor core's fp32 accumulation are less exact than k2b_v4's fp32 FMAs of
// the same operands, and MU amplifies the difference over 200 iterations on a
// tensor without low-rank structure. A single update_a stayed within 3e-6 of
// fp64 (tools/probe_update_a.py). Kept for reference; the product keeps k2b_v4.
//
// K2b on tensor cores — the dense one-GPU A update (K in {16, 32}):
//
//   num_i = sum_t P_t[i] R_t^T + Q_t[i] R_t          (rescal.py:133-143)
//   A_i  <- A_i * num_i / (A_i M + m eps)            (rescal.py:144-145)
//
// i.e. a (n x 2mK) . (2mK x K) product streamed from the stored P_t = X_t A,
// Q_t = X_t^T A (fp32, K1 + k1_reduce), plus the next iteration's operand
// planes (A in fp32, A^T as bf16 hi / lo). It replaces k2b_v4, whose per-row
// fp32 FMAs from shared memory ran ~6x its HBM time at cfg3 (166 us for
// 134 MB of P / Q).
//
// mma.sync m16n8k8 TF32 with a 3-pass split (a_lo b_hi + a_hi b_lo +
// a_hi b_hi; hi = truncation to tf32, lo exact) in fp32, added to fp64
// accumulators every two slices — the sparse path's sp_numer_tc scheme
// (sparse.cuh) generalised to K = 32. Block = 128 rows (8 warps x one 16-row
// m-tile), lane (g, tq) owns rows g, g + 8 and columns 8 nt + 2 tq + {0, 1}.
// Persistent, two CTAs per SM: a ring of (row block, slice) stages -- the
// block's P_t and Q_t rows and the slice's per-lane TF32 fragments of
// [R_t^T ; R_t] (k2b_tc_wfrag) -- filled by bulk copies (cp.async.bulk,
// mbarrier complete_tx).
#pragma once

#include "k1_tc.cuh"
#include "rk_common.cuh"
#include "rk_kernels.cuh"
#include "sparse.cuh"

namespace rk {

template <int K>
struct K2bTc {
  static constexpr int RB = 128;                     // rows per block
  static constexpr int NT = K / 8;                   // n-tiles (8 output columns each)
  static constexpr int KS = K / 8;                   // k-steps of 8 per operand
  static constexpr int NS = K == 32 ? 2 : 3;        // ring stages (two CTAs per SM)
  static constexpr int PQ_BYTES = RB * K * 4;        // one of P_t / Q_t rows
  static constexpr int WF_F4 = 2 * KS * NT * 32;     // float4 fragments per slice
  static constexpr int WF_BYTES = WF_F4 * 16;
  static constexpr int STAGE = 2 * PQ_BYTES + WF_BYTES;
  static constexpr size_t smem = (size_t)NS * STAGE + K * K * sizeof(double) + NS * 8 + 128;
};

// Per-lane TF32 hi / lo fragments of W_t = R_t^T (pq 0) | R_t (pq 1) from
// W32 = [R_t^T ; R_t] (fp32, written by the k2f commit):
// Wf[t][pq][s][nt][lane] = {b0_hi, b1_hi, b0_lo, b1_lo}, lane = 4 g + tq,
// b0 = W[kc(s, tq)][8 nt + g], b1 = W[kc(s, tq) + 1][8 nt + g] with the
// k-column permutation kc(s, tq) = 16 (s / 2) + 4 tq + 2 (s % 2) that lets a
// lane read its A fragments of all k-steps as float4s of its own rows.
template <int K>
__global__ void __launch_bounds__(256) k2b_tc_wfrag(const Ctl* __restrict__ ctl, const float* __restrict__ W32,
                                                    float4* __restrict__ Wf, int M) {
  using C = K2bTc<K>;
  if (ctl->stop) return;
  const int t = blockIdx.x;
  for (int e = threadIdx.x; e < C::WF_F4; e += blockDim.x) {
    const int lane = e & 31, combo = e >> 5;  // combo = (pq * KS + s) * NT + nt
    const int nt = combo % C::NT, s = (combo / C::NT) % C::KS, pq = combo / (C::NT * C::KS);
    const int g = lane >> 2, tq = lane & 3;
    const int kc = 16 * (s >> 1) + 4 * tq + 2 * (s & 1);
    const float* W = W32 + ((size_t)t * 2 + pq) * K * K;
    const float b0 = W[kc * K + 8 * nt + g], b1 = W[(kc + 1) * K + 8 * nt + g];
    const uint32_t h0 = sp::tf32_rna(b0), h1 = sp::tf32_rna(b1);
    const uint32_t l0 = sp::tf32_rna(b0 - __uint_as_float(h0)), l1 = sp::tf32_rna(b1 - __uint_as_float(h1));
    Wf[(size_t)t * C::WF_F4 + e] =
        make_float4(__uint_as_float(h0), __uint_as_float(h1), __uint_as_float(l0), __uint_as_float(l1));
  }
}

template <int K>
__global__ void __launch_bounds__(256, 2) k2b_tc(Ctl* __restrict__ ctl, double* __restrict__ A64,
                                                 float* __restrict__ A32, __nv_bfloat16* __restrict__ ATh,
                                                 __nv_bfloat16* __restrict__ ATl, const float* __restrict__ P,
                                                 const float* __restrict__ Q, const float4* __restrict__ Wf,
                                                 const double* __restrict__ Mm, int N, int M, double eps_m) {
  static_assert(K == 16 || K == 32, "k2b_tc: K in {16, 32}");
  using C = K2bTc<K>;
  constexpr int NT = C::NT, KS = C::KS;
  pdl_entry();
  if (ctl->stop) return;
  extern __shared__ __align__(128) uint8_t ksm[];
  uint8_t* ring = ksm;
  double* Ms = reinterpret_cast<double*>(ksm + (size_t)C::NS * C::STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(Ms + K * K);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int nrb = (N + C::RB - 1) / C::RB;
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
    const int nr = min(C::RB, N - row0);
    uint8_t* st = ring + (size_t)(f % C::NS) * C::STAGE;
    const uint32_t bar = tc::smem_u32(&full[f % C::NS]);
    const uint32_t bytes = (uint32_t)nr * K * 4;
    tc::mbar_expect_tx(bar, 2 * bytes + C::WF_BYTES);
    sp::bulk_g2s(tc::smem_u32(st), P + ((size_t)t * N + row0) * K, bytes, bar);
    sp::bulk_g2s(tc::smem_u32(st + C::PQ_BYTES), Q + ((size_t)t * N + row0) * K, bytes, bar);
    sp::bulk_g2s(tc::smem_u32(st + 2 * C::PQ_BYTES), Wf + (size_t)t * C::WF_F4, C::WF_BYTES, bar);
  };
  if (tid == 0)
    for (int f = 0; f < C::NS - 1 && f < nstage; ++f) issue(f);
  double acc[NT][4];
  float c[NT][4];
  bool bad = false;
  for (int f = 0; f < nstage; ++f) {
    const int t = f % M;
    const int row0 = ((int)blockIdx.x + (f / M) * (int)gridDim.x) * C::RB;
    const int nr = min(C::RB, N - row0);
    if (tid == 0 && f + C::NS - 1 < nstage) issue(f + C::NS - 1);
    tc::mbar_wait(tc::smem_u32(&full[f % C::NS]), (uint32_t)((f / C::NS) & 1));
    if (t == 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int x = 0; x < 4; ++x) acc[nt][x] = 0.0;
    }
    if ((t & 1) == 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int x = 0; x < 4; ++x) c[nt][x] = 0.f;
    }
    const uint8_t* st = ring + (size_t)(f % C::NS) * C::STAGE;
    const float4* wf = reinterpret_cast<const float4*>(st + 2 * C::PQ_BYTES);
    const int r = warp * 16 + g;  // rows r, r + 8 of the block (rows >= nr were never loaded: finite junk, unused)
#pragma unroll
    for (int pq = 0; pq < 2; ++pq) {
      const float* S = reinterpret_cast<const float*>(st + pq * C::PQ_BYTES);
#pragma unroll
      for (int hh = 0; hh < K / 16; ++hh) {
        const float4 x0 = *reinterpret_cast<const float4*>(S + r * K + 16 * hh + 4 * tq);
        const float4 x1 = *reinterpret_cast<const float4*>(S + (r + 8) * K + 16 * hh + 4 * tq);
#pragma unroll
        for (int ss = 0; ss < 2; ++ss) {
          const int s = 2 * hh + ss;
          const float v[4] = {ss ? x0.z : x0.x, ss ? x1.z : x1.x, ss ? x0.w : x0.y, ss ? x1.w : x1.y};
          uint32_t ah[4], al[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {  // hi = truncation to tf32 (one LOP), lo exact
            ah[q] = __float_as_uint(v[q]) & 0xffffe000u;
            al[q] = __float_as_uint(v[q] - __uint_as_float(ah[q]));
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const float4 b = wf[((pq * KS + s) * NT + nt) * 32 + lane];
            sp::mma_tf32(c[nt], al, __float_as_uint(b.x), __float_as_uint(b.y));
            sp::mma_tf32(c[nt], ah, __float_as_uint(b.z), __float_as_uint(b.w));
            sp::mma_tf32(c[nt], ah, __float_as_uint(b.x), __float_as_uint(b.y));
          }
        }
      }
    }
    if ((t & 1) || t == M - 1) {  // fp32 over <= 2 slices, then fp64
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int x = 0; x < 4; ++x) acc[nt][x] += (double)c[nt][x];
    }
    if (t == M - 1) {
      // A update of this row block: lane (g, tq) holds rows r (c0, c1) and
      // r + 8 (c2, c3) at columns 8 nt + 2 tq + {0, 1}. A row is read and
      // written only by the four lanes of one quad (same warp): a warp
      // barrier orders each row's reads before its writes.
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = r + 8 * h;
        const bool ok = rr < nr;
        const int i = row0 + (ok ? rr : 0);
        double* Ai = A64 + (size_t)i * K;
        double out[NT][2];
        if (ok) {
          double deno[NT][2];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) deno[nt][0] = deno[nt][1] = eps_m;
#pragma unroll 4
          for (int d = 0; d < K; ++d) {
            const double a = Ai[d];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const double2 mv = *reinterpret_cast<const double2*>(Ms + d * K + 8 * nt + 2 * tq);
              deno[nt][0] = fma(a, mv.x, deno[nt][0]);
              deno[nt][1] = fma(a, mv.y, deno[nt][1]);
            }
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const double2 av = *reinterpret_cast<const double2*>(Ai + 8 * nt + 2 * tq);
            out[nt][0] = av.x * acc[nt][2 * h] / deno[nt][0];
            out[nt][1] = av.y * acc[nt][2 * h + 1] / deno[nt][1];
            bad |= !(isfinite(out[nt][0]) && isfinite(out[nt][1]));
          }
        }
        __syncwarp();
        if (ok) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int col = 8 * nt + 2 * tq;
            *reinterpret_cast<double2*>(Ai + col) = make_double2(out[nt][0], out[nt][1]);
            *reinterpret_cast<float2*>(A32 + (size_t)i * K + col) = make_float2((float)out[nt][0], (float)out[nt][1]);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              __nv_bfloat16 hi, lo;
              split_bf16(out[nt][j], hi, lo);
              ATh[(size_t)(col + j) * N + i] = hi;
              ATl[(size_t)(col + j) * N + i] = lo;
            }
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

}  // namespace rk
