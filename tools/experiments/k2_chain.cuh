// EXPERIMENT (not built into librescal_b200.so): measured slower than the
// five separate kernels it replaces, so the product keeps those. Round-2 data
// (B200, graph-replayed iterations, tools/experiments/chain_probe.py,
// profiles/r02_chain_experiment.json):
//   it/s chain vs separate: cfg1 27.4k vs 32.0k, cfg2 1325 vs 1338,
//   cfg5 689 vs 695, n=2048/k=32 7.6k vs 9.1k, cfg3 78.1 vs 78.7.
//   Phase edges of one launch (us from block 0's entry), cfg2:
//   A end 30.7, barrier 1 exit 33.6, B end 50.5, barrier 2 exit 53.8,
//   C end 72.2 -- each grid barrier costs ~2.5-3 us, more than a kernel
//   boundary inside a CUDA graph, and every phase stays latency-bound with
//   fewer co-resident warps than the standalone kernel it replaces.
// It compiled against the phase bodies the standalone kernels share
// (tc::k1_reduce_p4 / k1_reduce_q4, sp::sp_gram_tc_body, k2f_body,
// k2b_v4_block) and was bit-identical to them (GPU test, round 2).
//
// k2_chain — the k-wide part of one MU iteration in ONE persistent launch
// (single GPU, dense, K in {16, 32}), after the K1 slice contraction:
//
//   rescal.py:124     G = A^T A
//   rescal.py:129     S_t = A^T P_t                (P_t = X_t A from K1's partials)
//   rescal.py:130-132 R_t <- R_t * S_t / (G R_t G + eps)
//   rescal.py:137-143 M = sum_t R_t^T G R_t + R_t G R_t^T
//   rescal.py:133-145 A <- A * (sum_t P_t R_t^T + Q_t R_t) / (A M + m eps)
//
// It replaces five launches (k1_reduce, sp_gram_tc_k, sp_gram_reduce,
// k2f_fused_t, k2b_v4) with the SAME arithmetic in the same order (the phase
// bodies are shared with those kernels, so the factors are bit-identical)
// and two grid-wide barriers:
//
//   phase A  every block: reduce the P rows of its own (slice, row chunk)
//            G/S groups from K1's strip partials, then the Q rows (grid
//            stride), then its G / S_t partials on tensor cores (mma.sync
//            TF32 3-pass, fp64 per 32 rows) -- the P rows it needs were
//            reduced by itself a moment before, so no grid barrier between
//   barrier
//   phase B  block t < m: sums the chunk partials of G and S_t in chunk
//            order, then the per-slice core update (k2f); the last block
//            (atomic ticket) keeps the trace / tolerance / commit R <- R'
//            and forms M
//   barrier
//   phase C  every block: A update + the next iteration's operand planes for
//            its row blocks (k2b_v4 body, coherent loads)
//
// Co-residency of all blocks (the barrier's requirement) is guaranteed by a
// cooperative launch sized from the occupancy calculator.
#pragma once

#include "k1_tc.cuh"
#include "rk_kernels.cuh"
#include "sparse.cuh"

namespace rk {

struct ChainArgs {
  Ctl* ctl;
  // phase A
  const float* Ppart;
  const float* Qpart;
  const int* slot_first;
  const int* slot_count;
  float* P;
  float* Q;
  int NR, NC, M, c, nstrips;
  float* A32;
  int rows_valid, gchunks;
  double* gpart;  // [(M+1)][gchunks][K*K]
  // phase B
  double* red;  // reduced [G, S_1..S_m]
  double* gsx;  // [M][K*K]: block t's copy of G
  double *R, *Rnext, *Mt, *Mm, *tt;
  const double* rres;
  int nres;
  double* trace;
  double eps;
  unsigned* ticket;  // k2f's last-block counter (self-resetting)
  float* W32;
  // phase C
  double* A64;
  __nv_bfloat16 *ATh, *ATl;
  int tg;
  double eps_m;
  unsigned* bar;  // [2]: arrival count, generation (self-resetting)
  int sleep_ns;   // barrier poll back-off
  unsigned long long* stamps;  // diagnostics: [6] globaltimer at the phase edges (null: off)
};

RK_DEV unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Grid-wide barrier (all blocks co-resident): arrive on a counter, the last
// arrival resets it and bumps the generation the others spin on.
RK_DEV void chain_grid_sync(unsigned* bar, unsigned nblocks, int sleep_ns) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    const unsigned gen = *vgen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen)
        if (sleep_ns) __nanosleep(sleep_ns);
    }
    __threadfence();
  }
  __syncthreads();
}

template <int K, int RPT>
__global__ void __launch_bounds__(256) k2_chain(ChainArgs a) {
  static_assert(K == 16 || K == 32, "k2_chain: K in {16, 32}");
  if (a.ctl->stop) return;  // set before this launch: every block takes the same exit
  if (a.stamps && threadIdx.x == 0 && blockIdx.x == 0) a.stamps[0] = globaltimer_ns();
  extern __shared__ __align__(16) float csm[];
  const int bid = blockIdx.x, nblk = gridDim.x, tid = threadIdx.x;
  const int M = a.M;
  constexpr int KK = K * K, K4 = K / 4;

  // ---------------- phase A: P / Q reduce + G / S_t partials ----------------
  {
    const int n = a.rows_valid, nchunk = a.gchunks;
    const int rpc = (n + nchunk - 1) / nchunk;
    // (a) the P rows of this block's (slot >= 1, chunk) groups -- exactly the
    //     rows its sp_gram_tc_body items below read (groups bid, bid + nblk, ...)
    for (int sc = bid; sc < (M + 1) * nchunk; sc += nblk) {
      const int slot = sc / nchunk, chunk = sc - slot * nchunk;
      if (slot == 0) continue;
      const int r0 = chunk * rpc, r1 = min(n, r0 + rpc);
      for (int e = tid; e < (r1 - r0) * K4; e += 256)
        tc::k1_reduce_p4(a.Ppart, a.P, a.NR, K, M, a.nstrips, slot - 1, r0 + e / K4, e % K4);
    }
    // (b) the padding rows of P and all of Q, grid stride
    const int64_t gtid = (int64_t)bid * 256 + tid, gstr = (int64_t)nblk * 256;
    const int64_t npad = (int64_t)M * (a.NR - n) * K4;
    for (int64_t e = gtid; e < npad; e += gstr) {
      const int q4 = (int)(e % K4);
      const int64_t ti = e / K4;
      tc::k1_reduce_p4(a.Ppart, a.P, a.NR, K, M, a.nstrips, (int)(ti / (a.NR - n)), n + (int)(ti % (a.NR - n)),
                       q4);
    }
    const int64_t nq = (int64_t)M * a.NC * K4;
    for (int64_t e = gtid; e < nq; e += gstr) {
      const int q4 = (int)(e % K4);
      const int64_t tj = e / K4;
      tc::k1_reduce_q4(a.Qpart, a.slot_first, a.slot_count, a.Q, a.NC, K, a.c, a.nstrips, (int)(tj / a.NC),
                       (int)(tj % a.NC), q4);
    }
    __threadfence();
    __syncthreads();
    // (c) G / S_t chunk partials (cp.async.cg reads of P go through L2)
    sp::sp_gram_tc_body<K>(a.A32, a.P, n, a.NR, M, nchunk, a.gpart, nullptr, 0, bid, nblk, csm);
  }
  if (a.stamps && tid == 0) atomicMax(a.stamps + 1 + 2 * 0, globaltimer_ns());
  chain_grid_sync(a.bar, nblk, a.sleep_ns);
  if (a.stamps && tid == 0 && bid == 0) a.stamps[2] = globaltimer_ns();

  // ---------------- phase B: per-slice core update, M, commit ---------------
  if (bid < M) {
    const int t = bid, nchunk = a.gchunks;
    double* gsG = a.gsx + (size_t)t * KK;
    for (int e = tid; e < KK; e += 256) {
      const double g = sp::sum_chunks(a.gpart + e, nchunk, KK);
      const double s = sp::sum_chunks(a.gpart + (size_t)(1 + t) * nchunk * KK + e, nchunk, KK);
      gsG[e] = g;
      if (t == 0) a.red[e] = g;
      a.red[(size_t)(1 + t) * KK + e] = s;
    }
    __syncthreads();
    k2f_body<K>(a.ctl, gsG, a.red + (size_t)(1 + t) * KK, a.R, a.Rnext, a.Mt, a.Mm, a.tt, a.rres, a.nres,
                a.trace, K, M, a.eps, 0, nullptr, a.ticket, a.W32, reinterpret_cast<double*>(csm), t);
  }
  if (a.stamps && tid == 0) atomicMax(a.stamps + 3, globaltimer_ns());
  chain_grid_sync(a.bar, nblk, a.sleep_ns);
  if (a.stamps && tid == 0 && bid == 0) a.stamps[4] = globaltimer_ns();

  // ---------------- phase C: A update + operand planes ----------------------
  if (*reinterpret_cast<volatile int*>(&a.ctl->stop)) return;  // tolerance / non-finite: same on every block
  constexpr int RB = RPT * (256 / K);
  const int nrb = (a.NR + RB - 1) / RB;
  for (int rbi = bid; rbi < nrb; rbi += nblk)
    k2b_v4_block<K, RPT, true>(a.ctl, a.A64, a.A32, a.ATh, a.ATl, a.P, a.Q, a.W32, a.Mm,
                               a.NR, M, a.tg, a.eps_m, rbi, csm);
  if (a.stamps && tid == 0) atomicMax(a.stamps + 5, globaltimer_ns());
}

// fused-kernel k2b staging: slices per group so that its shared memory stays
// within the G / S stage buffers (SpGramTc::smem)
inline int k2_chain_tg(int K, int M, int64_t N) {
  const int RB = k2b_v4_rb(K, N);
  const size_t per = (size_t)(2 * K * K + 2 * RB * K) * sizeof(float);
  return (int)std::max<size_t>(1, std::min<size_t>((size_t)M, sp::SpGramTc::smem / per));
}

inline size_t k2_chain_smem(int K, int M, int64_t N) {
  const int RB = k2b_v4_rb(K, N);
  const size_t k2b = (size_t)k2_chain_tg(K, M, N) * (2 * K * K + 2 * RB * K) * sizeof(float);
  const size_t k2f = (size_t)5 * K * K * sizeof(double);
  return std::max(std::max(sp::SpGramTc::smem, k2b), k2f);
}

}  // namespace rk
