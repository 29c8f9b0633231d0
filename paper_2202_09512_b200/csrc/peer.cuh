// Peer-memory grid exchange (NVLink / NVSwitch, one process per GPU).
//
// Replaces the per-iteration NCCL calls of the p_r x p_c grid schedule
// (rescal_b200.cu grid_allreduce_parts / launch_k2b) with
// stores straight into the peers' memory, fused into the kernels that produce
// the data:
//   peer_allreduce  : [G, S_1..S_m, residual] partial -> slot `rank` of every
//                     peer; each CTA then sums one chunk of the p slots in rank
//                     order (identical bytes on every rank -> R stays replicated,
//                     the invariant of test_dist_rescal.py:65-78)
//   k2b_u4_peer     : numerator rows U_I = sum_t P_t R_t^T (row set) and
//                     U_J = sum_t Q_t R_t (column set) computed and written
//                     directly into the owning rank's receive slot (the
//                     reduce-scatter of dist_rescal.py:150-158 without a
//                     separate collective)
//   apply_peer      : owner sums its slots in fixed order, updates its A piece
//                     (rescal.py:144-145) and writes the new rows into the row
//                     and column peers' receive slots (the all-gather)
//   emit_peer       : assembles A_row / A_col from the received pieces and
//                     emits the next iteration's operand planes
// Each rank owns one IPC-shared arena: flags | red slots | rxI | rxJ | rxA_row |
// rxA_col, every data region double-buffered by epoch parity (a rank can run
// at most one exchange ahead of a peer). Completion is signalled per (kind,
// parity, source) with st.release.sys of the epoch after a system fence;
// receivers poll with ld.acquire.sys (bounded by a 20 s timeout that raises
// Ctl::peer_err instead of hanging the device). Multi-CTA producers signal
// from the last CTA (atomic ticket), after every CTA's __threadfence_system().
#pragma once

#include "rk_kernels.cuh"

namespace rk {
namespace peer {

constexpr int kMaxP = 16;
enum Kind { F_RED = 0, F_I = 1, F_J = 2, F_AR = 3, F_AC = 4, F_KINDS = 5 };
constexpr size_t kFlagBytes = 4096;  // F_KINDS * 2 * kMaxP * 4 <= 4096

struct Args {
  char* base[kMaxP];  // arena of every rank (own included), mapped in this process
  unsigned* ep;       // local: [0] all-reduce epoch [1] numerator/A epoch; [4..7] tickets
  Ctl* ctl;
  int p, pr, pc, rank, gi, gj, K, L;  // L = (m+1) K^2 + 1 doubles per red slot
  long long b;                        // piece rows
  long long off_red, off_rxI, off_rxJ, off_rxAr, off_rxAc;  // byte offsets in an arena
};

RK_DEV unsigned* flag_at(const Args& a, int dst, int kind, int par, int src) {
  return reinterpret_cast<unsigned*>(a.base[dst]) + ((kind * 2 + par) * kMaxP + src);
}
RK_DEV void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
RK_DEV unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
RK_DEV unsigned ld_volatile(const unsigned* p) {
  unsigned v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
RK_DEV uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// flag values only grow; (int)(v - e) >= 0 tolerates a peer one epoch ahead
RK_DEV void wait_flag(const unsigned* f, unsigned e, Ctl* ctl) {
  if ((int)(ld_acquire_sys(f) - e) >= 0) return;
  const uint64_t t0 = global_ns();
  while ((int)(ld_acquire_sys(f) - e) < 0) {
    if (*(volatile int*)&ctl->peer_err) return;
    if (global_ns() - t0 > 20000000000ull) {
      atomicExch(&ctl->peer_err, 1);
      return;
    }
    __nanosleep(100);
  }
}
// threads [0, pc) wait for the row peers' flags, [32, 32 + pr) for the column peers'
RK_DEV void wait_row_col(const Args& a, int kind_row, int kind_col, int par, unsigned e) {
  const int t = threadIdx.x;
  if (t < a.pc) wait_flag(flag_at(a, a.rank, kind_row, par, a.gi * a.pc + t), e, a.ctl);
  if (t >= 32 && t < 32 + a.pr) wait_flag(flag_at(a, a.rank, kind_col, par, (t - 32) * a.pc + a.gj), e, a.ctl);
  __syncthreads();
}
// last-CTA ticket: true in exactly one thread of the last CTA to finish
RK_DEV bool last_cta(unsigned* ticket, unsigned nctas) {
  __shared__ unsigned s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned t = atomicAdd(ticket, 1u);
    s_last = (t == nctas - 1) ? 1u : 0u;
    if (s_last) {
      *ticket = 0u;
      __threadfence_system();
    }
  }
  __syncthreads();
  return threadIdx.x == 0 && s_last;
}

// grid = p CTAs. CTA d sends the local partial to rank d, then sums chunk d.
__global__ void __launch_bounds__(512) peer_allreduce(Args a, double* __restrict__ red, int len,
                                                      const double* __restrict__ rpart, int nr) {
  __shared__ double scratch[32];
  const int d = blockIdx.x, tid = threadIdx.x;
  const unsigned e = a.ep[0] + 1u;
  const int par = (int)(e & 1u);
  double acc = 0.0;
  for (int i = tid; i < nr; i += blockDim.x) acc += rpart[i];
  acc = block_sum(acc, scratch);
  double* dst = reinterpret_cast<double*>(a.base[d] + a.off_red) + ((size_t)par * a.p + a.rank) * a.L;
  for (int i = tid; i < len; i += blockDim.x) dst[i] = red[i];
  if (tid == 0) dst[len] = acc;
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    st_release_sys(flag_at(a, d, F_RED, par, a.rank), e);
    atomicAdd(&a.ep[4], 1u);  // local read barrier: this CTA is done reading red
  }
  if (tid < a.p) wait_flag(flag_at(a, a.rank, F_RED, par, tid), e, a.ctl);
  if (tid == 0) {
    const uint64_t t0 = global_ns();
    while (ld_volatile(&a.ep[4]) < (unsigned)a.p && !*(volatile int*)&a.ctl->peer_err) {
      if (global_ns() - t0 > 20000000000ull) atomicExch(&a.ctl->peer_err, 1);
    }
    __threadfence();
  }
  __syncthreads();
  const double* slots = reinterpret_cast<const double*>(a.base[a.rank] + a.off_red) + (size_t)par * a.p * a.L;
  const int chunk = (a.L + a.p - 1) / a.p;
  const int i1 = min(a.L, (d + 1) * chunk);
  for (int i = d * chunk + tid; i < i1; i += blockDim.x) {
    double s = 0.0;
    for (int src = 0; src < a.p; ++src) s += slots[(size_t)src * a.L + i];
    red[i] = s;  // red[len] = the summed residual scalar
  }
  if (last_cta(&a.ep[5], gridDim.x)) {
    a.ep[4] = 0u;
    a.ep[0] = e;
    __threadfence();
  }
}

// Numerator rows, blockIdx.y = 0: U_I rows of the row set (P side), 1: U_J rows
// of the column set (Q side), written into the owner's rxI / rxJ slot.
template <int K>
__global__ void __launch_bounds__(256) k2b_u4_peer(const Ctl* __restrict__ ctl, const float* __restrict__ P,
                                                   const float* __restrict__ Q, const float* __restrict__ W32,
                                                   int NR, int NC, int M, int tg, Args a) {
  constexpr int TR = 256 / K;
  const int which = blockIdx.y;
  const int N = which ? NC : NR;
  const unsigned e = a.ep[1] + 1u;
  const int par = (int)(e & 1u);
  const int rbase = blockIdx.x * 2 * TR;
  if (!ctl->stop && rbase < N) {
    double n0, n1;
    k2b_u4_rows<K>(which ? Q : P, W32, which, N, M, tg, rbase, n0, n1);
    const int rl = threadIdx.x / K, c = threadIdx.x - rl * K;
    const long long nvalid = (long long)(which ? a.pr : a.pc) * a.b;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long i = rbase + rl + h * TR;
      if (i >= N || i >= nvalid) continue;
      const int slot = (int)(i / a.b);
      const long long r = i - (long long)slot * a.b;
      double* dst;
      if (which == 0)  // owner (gi, slot), my slot there = gj
        dst = reinterpret_cast<double*>(a.base[a.gi * a.pc + slot] + a.off_rxI) +
              (((size_t)par * a.pc + a.gj) * a.b + r) * K;
      else  // owner (slot, gj), my slot there = gi
        dst = reinterpret_cast<double*>(a.base[slot * a.pc + a.gj] + a.off_rxJ) +
              (((size_t)par * a.pr + a.gi) * a.b + r) * K;
      dst[c] = h ? n1 : n0;
    }
  }
  if (last_cta(&a.ep[6], gridDim.x * gridDim.y)) {
    for (int jj = 0; jj < a.pc; ++jj) st_release_sys(flag_at(a, a.gi * a.pc + jj, F_I, par, a.rank), e);
    for (int ii = 0; ii < a.pr; ++ii) st_release_sys(flag_at(a, ii * a.pc + a.gj, F_J, par, a.rank), e);
    a.ep[1] = e;
    __threadfence();
  }
}

// Sparse grid (K = 16): the numerator rows U_I / U_J come from sp_numer_tc
// into local buffers; this pushes them into the owners' rxI / rxJ slots (the
// reduce-scatter's data movement, summed at the owner in fixed order) and
// signals like k2b_u4_peer. A stopped run still signals (peers never wait on
// a rank that skipped).
__global__ void __launch_bounds__(256) push_u_peer(const Ctl* __restrict__ ctl, const double* __restrict__ UI,
                                                   const double* __restrict__ UJ, Args a) {
  const unsigned e = a.ep[1] + 1u;
  const int par = (int)(e & 1u);
  const int K = a.K, K2 = K / 2;
  if (!ctl->stop) {
    const long long nI = (long long)a.pc * a.b * K2, nJ = (long long)a.pr * a.b * K2;  // double2 units
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < nI + nJ;
         x += (long long)gridDim.x * blockDim.x) {
      const bool jside = x >= nI;
      const long long el = jside ? x - nI : x;
      const long long i = el / K2;
      const int c2 = (int)(el - i * K2);
      const int slot = (int)(i / a.b);
      const long long r = i - (long long)slot * a.b;
      const double2 v = reinterpret_cast<const double2*>(jside ? UJ : UI)[el];
      double* dst;
      if (!jside)
        dst = reinterpret_cast<double*>(a.base[a.gi * a.pc + slot] + a.off_rxI) +
              (((size_t)par * a.pc + a.gj) * a.b + r) * K;
      else
        dst = reinterpret_cast<double*>(a.base[slot * a.pc + a.gj] + a.off_rxJ) +
              (((size_t)par * a.pr + a.gi) * a.b + r) * K;
      reinterpret_cast<double2*>(dst)[c2] = v;
    }
  }
  if (last_cta(&a.ep[6], gridDim.x)) {
    for (int jj = 0; jj < a.pc; ++jj) st_release_sys(flag_at(a, a.gi * a.pc + jj, F_I, par, a.rank), e);
    for (int ii = 0; ii < a.pr; ++ii) st_release_sys(flag_at(a, ii * a.pc + a.gj, F_J, par, a.rank), e);
    a.ep[1] = e;
    __threadfence();
  }
}

// Owner: A_own <- A_own * (sum_j rxI + sum_i rxJ) / (A_own M + m eps), sent to
// the row peers' rxA_row[gj] and the column peers' rxA_col[gi]. A stopped run
// re-sends the unchanged rows (the peers' copies stay what they were).
__global__ void __launch_bounds__(kThreads) apply_peer(Ctl* __restrict__ ctl, const double* __restrict__ Aown,
                                                       const double* __restrict__ Mm, int K, double eps_m,
                                                       Args a) {
  const unsigned e = a.ep[1];
  const int par = (int)(e & 1u);
  const bool stopped = ctl->stop != 0;
  wait_row_col(a, F_I, F_J, par, e);
  const int rpb = kThreads / K;
  const int r = threadIdx.x / K, c = threadIdx.x - r * K;
  const long long i = (long long)blockIdx.x * rpb + r;
  if (r < rpb && i < a.b) {
    const double* Ai = Aown + (size_t)i * K;
    double anew = Ai[c];
    if (!stopped) {
      const double* rxI = reinterpret_cast<const double*>(a.base[a.rank] + a.off_rxI);
      const double* rxJ = reinterpret_cast<const double*>(a.base[a.rank] + a.off_rxJ);
      double sI = 0.0, sJ = 0.0;
      for (int jj = 0; jj < a.pc; ++jj) sI += rxI[(((size_t)par * a.pc + jj) * a.b + i) * K + c];
      for (int ii = 0; ii < a.pr; ++ii) sJ += rxJ[(((size_t)par * a.pr + ii) * a.b + i) * K + c];
      double deno = eps_m;
      for (int dd = 0; dd < K; ++dd) deno = fma(Ai[dd], Mm[dd * K + c], deno);
      anew = Ai[c] * (sI + sJ) / deno;
      // no stop here: only this rank would see it and its peers would wait
      // for its next exchange. The value travels to every peer with the
      // piece, turns the next replicated core update non-finite on ALL
      // ranks, and there every rank stops at the same iteration.
      if (!isfinite(anew)) ctl->nonfinite = 1;
    }
    for (int jj = 0; jj < a.pc; ++jj)
      reinterpret_cast<double*>(a.base[a.gi * a.pc + jj] + a.off_rxAr)[(((size_t)par * a.pc + a.gj) * a.b + i) * K + c] = anew;
    for (int ii = 0; ii < a.pr; ++ii)
      reinterpret_cast<double*>(a.base[ii * a.pc + a.gj] + a.off_rxAc)[(((size_t)par * a.pr + a.gi) * a.b + i) * K + c] = anew;
  }
  if (last_cta(&a.ep[7], gridDim.x)) {
    for (int jj = 0; jj < a.pc; ++jj) st_release_sys(flag_at(a, a.gi * a.pc + jj, F_AR, par, a.rank), e);
    for (int ii = 0; ii < a.pr; ++ii) st_release_sys(flag_at(a, ii * a.pc + a.gj, F_AC, par, a.rank), e);
  }
}

// A_row = [rxA_row slots], A_col = [rxA_col slots] (fp64 masters) + fp32 copies and
// transposed bf16 hi/lo operand planes (as emit_operands).
__global__ void __launch_bounds__(kThreads) emit_peer(Args a, double* __restrict__ Arow, int NR,
                                                      float* __restrict__ A32row, __nv_bfloat16* __restrict__ AThr,
                                                      __nv_bfloat16* __restrict__ ATlr, double* __restrict__ Acol,
                                                      int NC, float* __restrict__ A32col,
                                                      __nv_bfloat16* __restrict__ AThc, __nv_bfloat16* __restrict__ ATlc) {
  const unsigned e = a.ep[1];
  const int par = (int)(e & 1u);
  wait_row_col(a, F_AR, F_AC, par, e);
  const int K = a.K;
  const double* rxr = reinterpret_cast<const double*>(a.base[a.rank] + a.off_rxAr) + (size_t)par * a.pc * a.b * K;
  const double* rxc = reinterpret_cast<const double*>(a.base[a.rank] + a.off_rxAc) + (size_t)par * a.pr * a.b * K;
  const int64_t nr = (int64_t)a.pc * a.b * K, nc = (int64_t)a.pr * a.b * K;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nr + nc; x += (int64_t)gridDim.x * blockDim.x) {
    const bool col = x >= nr;
    const int64_t el = col ? x - nr : x;
    const int i = (int)(el / K), c = (int)(el - (int64_t)i * K);
    const double v = col ? rxc[el] : rxr[el];
    __nv_bfloat16 hi, lo;
    split_bf16(v, hi, lo);
    if (col) {
      Acol[el] = v;
      A32col[el] = (float)v;
      if (AThc == nullptr) continue;  // sparse engine: fp32 copies only
      AThc[(size_t)c * NC + i] = hi;
      ATlc[(size_t)c * NC + i] = lo;
    } else {
      Arow[el] = v;
      A32row[el] = (float)v;
      if (AThr == nullptr) continue;
      AThr[(size_t)c * NR + i] = hi;
      ATlr[(size_t)c * NR + i] = lo;
    }
  }
}

}  // namespace peer
}  // namespace rk
