// K1 — tcgen05 dual slice contraction for the RESCAL MU iteration (sm_100a).
//
// Computes, for every slice t, P_t = X_t A and Q_t = X_t^T A in ONE pass over
// X (reference: rescal.py:128 X_t A and rescal.py:134-135 X_t^T (A R_t), the
// latter restructured as (X_t^T A) R_t so both products read the same X tile;
// SURVEY.md App. C). Split precision 3xBF16: X = Xh + Xl and A = Ah + Al are
// bf16 pairs; each product accumulates Xh*Ah + Xh*Al + Xl*Ah in fp32 TMEM.
//
// Work decomposition (persistent, one CTA per SM):
//   tile   = 128 x 128 block of one slice (rows i, cols j)
//   strip  = `c` consecutive column tiles (W = 128c columns)
//   item   = (t, strip, row-block rb): the c tiles of one row block in a strip
// Each CTA owns a contiguous range of items (balanced by tile count). Within
// an item the P accumulator (128 rows x K) lives in TMEM (double buffered);
// the c Q accumulators (one per column tile, 128 x K each) live in TMEM
// across the run of items the CTA has in the same (t, strip).
// Rotating Q drains (accuracy): the tensor core's fp32 accumulation loses
// ~1 ulp per accumulate step in one direction, so the relative error of a
// TMEM sum grows LINEARLY with its length (Q at n = 32768 summed over whole
// runs: 5.7e-5 with ~76-row-block runs; P, 12 tiles per item: 5e-6). So
// after the item of row block rb, Q tile (rb mod c) is drained — its TMEM
// sum added into the run's slot in fp32 (round-to-nearest) and restarted:
// every TMEM sum spans at most c row blocks, and one 16 KB tile leaves per
// item (like P). The MMAs reuse that tile only c - 1 tiles later, so the
// drain never stalls the tensor pipe (a drain of all c tiles at once costs
// ~6 us of stalled MMA per drain). At the end of a run all tiles drain.
// The slot (CTA-private, one per (CTA, run)) is read back by later drains:
// stored evict-last under an L2 set-aside. The CTA's final drain writes a
// fresh slot (a read-back there would sit on the kernel's tail). On by
// default (period args.qrot = 1, K <= 32): without it the cfg3-shape factors
// leave north_star's 1e-4 within a few MU iterations.
// Strip groups (args.grp = 2 or 4): the CTAs of a group share a strip of up
// to grp * c tiles, each accumulating its share of P in TMEM; the last to
// arrive per item sums the members' tiles (L2 scratch, member order) and
// writes the strip's one P partial -- 1/grp of the partial traffic.
//   P partial  -> Ppart[strip][t][row block][K/4][128] float4 (one writer per (t,strip,row))
//   Q partial  -> Qpart[slot][tile][K/4][128] float4
// k1_reduce sums the partials in a fixed order (deterministic, no atomics).
//
// Warp roles (192 threads): w0 TMA producer, w1 TMEM alloc + MMA issuer,
// w2..w5 epilogue (TMEM -> registers -> global), lane quadrant = warp % 4.
#pragma once

#include <cuda.h>

#include "rk_common.cuh"

namespace rk {
namespace tc {

constexpr int kTile = 128;
constexpr int kThreads = 192;
constexpr uint32_t kXBox = 128 * 64 * 2;  // one 128-row x 64-col bf16 box = 16 KB
constexpr int kMaxC = 16;                 // max column tiles per strip (TMEM: 512 / 32)

struct K1Args {
  int NR, NC, K, M;
  int c;          // tiles per strip
  int nstrips;
  int nrb;        // NR / 128 row blocks
  int ncb;        // NC / 128 column tiles
  int qrot;       // rotating Q drains: one tile every qrot items (0 = only at run ends)
  int grp;        // CTAs per strip group (1, 2 or 4; k1_tc.cuh "Strip groups")
  int sw;         // column tiles per strip (c, or <= grp * c with groups)
  float* Pscr;    // groups: [ngroups][kPairSlots][grp][K/4][128] float4, the members' P tiles
  unsigned* pflag;  // groups: [ngroups][kPairWords] tickets / ready / done / exit counters
  float* Ppart;   // [nstrips][M][NR/128][K/4][128] float4
  float* Qpart;   // [nslots][c][K/4][128] float4
  const int* cta_begin;  // [grid + 1] item ranges
  const int* cta_slot;   // [grid] first Q slot of the CTA
  const Ctl* ctl;
  int skip_if_stopped;
};

// ------------------------------- PTX helpers -------------------------------
RK_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

RK_DEV void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

RK_DEV void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

RK_DEV void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

RK_DEV void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

RK_DEV void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

RK_DEV void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// One lane of a converged warp (elect.sync). Issuing tcgen05.mma from an
// elected lane of a warp-uniform loop keeps the descriptors in uniform
// registers; issuing from an `if (lane == 0)` region instead makes ptxas wrap
// every UTCHMMA in an ELECT / BRA.U.ANY waterfall loop (measured ~20 cycles
// more per MMA, tools/umma_bench.cu).
RK_DEV bool elect_one() {
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

// warp index as a value ptxas can prove warp-uniform
RK_DEV int warp_id_uniform() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }

RK_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
RK_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

RK_DEV void tc_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}

// D[tmem] (+)= A[smem desc] * B[smem desc], kind::f16 (bf16 in, fp32 accum)
RK_DEV void tc_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                   uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 16 columns of 32-bit: thread = lane, 16 consecutive columns
RK_DEV void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor, SWIZZLE_128B, sm100 version bits.
RK_DEV uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor: kind::f16, A/B = BF16, D = F32, M = 128, N = n.
RK_DEV uint32_t idesc_bf16(int n, int a_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn_major << 15) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// item -> (t, strip, rb); items are ordered (t, strip, rb)
RK_DEV void decode_item(int item, int nstrips, int nrb, int& t, int& s, int& rb) {
  rb = item % nrb;
  int ts = item / nrb;
  s = ts % nstrips;
  t = ts / nstrips;
}

// the Q tile drained after row block rb (-1: none): tile (rb / p) mod c after
// every p-th row block (k1_plan mirrors this on the host)
__host__ __device__ inline int k1_rot_tile(int rb, int p, int c) {
  return p > 0 && rb % p == p - 1 ? (rb / p) % c : -1;
}

RK_DEV int strip_tiles(int s, int nstrips, int c, int ncb) {
  return s == nstrips - 1 ? ncb - c * (nstrips - 1) : c;
}

// The column tiles of strip s a CTA works on: all of them, or with a group
// of grp CTAs member q's share of a balanced split (the first cts mod grp
// members take one tile more).
__host__ __device__ inline void k1_half_tiles(int s, int nstrips, int sw, int ncb, int grp, int q, int& ct,
                                              int& toff) {
  const int cts = s == nstrips - 1 ? ncb - sw * (nstrips - 1) : sw;
  if (grp <= 1) {
    ct = cts;
    toff = 0;
    return;
  }
  const int base = cts / grp, rem = cts - base * grp;
  ct = base + (q < rem ? 1 : 0);
  toff = q * base + (q < rem ? q : rem);
}

RK_DEV void red_release_add_u32(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

RK_DEV unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

RK_DEV void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

RK_DEV void epi_bar() { asm volatile("bar.sync 2, 128;" ::: "memory"); }  // the 4 epilogue warps

constexpr int kPairSlots = 4;                   // scratch item slots per CTA group
constexpr int kMaxGrp = 4;                      // CTAs per strip group
constexpr int kPairWords = 3 * kPairSlots + 1;  // tickets, ready, done per slot + exit count

// ------------------------------- the kernel --------------------------------
// Operand merging: with MERGE_P the B operand of P is [A_hi ; A_lo] as ONE
// N = 2K MMA (X_hi is read once for both), the accumulator is 2K columns wide
// ([X_hi A_hi + X_lo A_hi | X_hi A_lo]) and the epilogue adds the halves.
// MERGE_Q does the same for Q. Halves the X_hi shared-memory reads of the
// MMA phase (the N = 16 MMAs are smem-read bound, not tensor bound).
//
// MMA count, not shared-memory bytes, paces the MMA phase: a kind::f16
// M = 128, K = 16 tcgen05.mma with N <= 64 costs ~45 cycles whatever N, A
// source (smem or TMEM) or major-ness (tools/umma_bench.cu,
// profiles/r02_umma_bench.log). Per 128 x 128 tile: 4 MMAs per k-step with
// both products merged (32 per tile), 5 with Q unmerged (40 per tile).
// MQ = merge Q; at K = 32 it costs TMEM (Q accumulators 2K wide: 6 column
// tiles per strip instead of 12, so twice the P partial traffic).
template <int K, bool MQ>
struct K1Cfg {
  static constexpr bool kMergeP = true;
  static constexpr bool kMergeQ = MQ;
  static constexpr int kPW = kMergeP ? 2 * K : K;  // TMEM columns per P buffer
  static constexpr int kQW = kMergeQ ? 2 * K : K;  // TMEM columns per Q accumulator
};

// Split stages: each 128 x 128 tile arrives as two sub-stages (the X hi
// plane with A_col's hi + lo boxes, then the X lo plane with A_col's hi
// boxes), so the shared memory holds 4 (K = 32) / 5 (K = 16) of them instead
// of 2 whole-tile stages: more bytes in flight per SM (round 2: cfg2 K1 0.976
// -> 0.997 of HBM, cfg3 11.90 -> 11.60-11.69 ms; profiles/r02_k1_split_stages).
// K = 48 / 64 (k from 33 to 64): the A boxes grow with K, so 3 / 2
// sub-stages fit next to the two A_row buffers (227 KB).
template <int K>
struct K1Stages {
  static constexpr uint32_t kABox = K * 128;
  static constexpr int kNSt = K == 16 ? 5 : K == 32 ? 4 : K == 48 ? 3 : 2;
  static constexpr uint32_t kSubBytes = 2 * kXBox + 4 * kABox;
};

// One Q tile's drain (epilogue thread = one TMEM lane / tile row): wait for
// the tile's commit, read its K columns, release the TMEM (q_empty), add the
// slot's earlier sum `old` when `add`, store the row (float4 column-major
// slot layout, stride 128 rows) with L2 policy `pol`.
template <int K, bool MQ>
RK_DEV void k1_drain_q(uint32_t taddr, uint32_t full_bar, uint32_t par, uint32_t empty_bar, int lane,
                       float4* dst, const float4 (&old)[K / 4], bool add, uint64_t pol) {
  mbar_wait(full_bar, par);
  tc_fence_after();
  float w[K];
#pragma unroll
  for (int h = 0; h < K / 16; ++h) tmem_ld16(taddr + 16 * h, w + 16 * h);
  if (MQ) {
    float w2[K];
#pragma unroll
    for (int h = 0; h < K / 16; ++h) tmem_ld16(taddr + K + 16 * h, w2 + 16 * h);
#pragma unroll
    for (int d = 0; d < K; ++d) w[d] += w2[d];
  }
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(empty_bar);
  if (add) {
#pragma unroll
    for (int h = 0; h < K / 4; ++h) {
      w[4 * h] += old[h].x;
      w[4 * h + 1] += old[h].y;
      w[4 * h + 2] += old[h].z;
      w[4 * h + 3] += old[h].w;
    }
  }
#pragma unroll
  for (int h = 0; h < K / 4; ++h)
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(dst + h * kTile),
                 "f"(w[4 * h]), "f"(w[4 * h + 1]), "f"(w[4 * h + 2]), "f"(w[4 * h + 3]), "l"(pol)
                 : "memory");
}

template <int K, bool MQ>
__global__ void __launch_bounds__(kThreads, 1)
    k1_tc_kernel(const __grid_constant__ CUtensorMap map_xh, const __grid_constant__ CUtensorMap map_xl,
                 const __grid_constant__ CUtensorMap map_rh, const __grid_constant__ CUtensorMap map_rl,
                 const __grid_constant__ CUtensorMap map_ch, const __grid_constant__ CUtensorMap map_cl,
                 K1Args args) {
  pdl_entry();
  // map_x*: the block's slices as a (M*NR) x NC bf16 matrix (hi / lo planes)
  // map_r*: A_row^T (K x NR) — B operand of Q = X^T A_row (indexed by row i)
  // map_c*: A_col^T (K x NC) — B operand of P = X A_col (indexed by col j)
  static_assert(K == 16 || K == 32 || K == 48 || K == 64, "tcgen05 path supports k_pad 16, 32, 48, 64");
  // rotating Q drains (read-back registers) only at K <= 32 (k1_qrot())
  constexpr bool kRot = K <= 32;
  constexpr bool kMergeP = K1Cfg<K, MQ>::kMergeP, kMergeQ = K1Cfg<K, MQ>::kMergeQ;
  constexpr int kPW = K1Cfg<K, MQ>::kPW, kQW = K1Cfg<K, MQ>::kQW;
  constexpr uint32_t kABox = K * 128;              // K rows x 64 bf16
  // A operand tiles hold the boxes as [hi b0][lo b0][hi b1][lo b1] so that
  // the hi and lo rows of one 64-column K chunk are contiguous (N = 2K view)
  // sub-stage: X0 X1 (one plane) | A_col boxes [hi b0][lo b0][hi b1][lo b1]
  constexpr int kNSt = K1Stages<K>::kNSt;
  constexpr uint32_t kStageX = 2 * kXBox;
  constexpr uint32_t kStageBytes = K1Stages<K>::kSubBytes;
  constexpr uint32_t kAIBytes = 4 * kABox;

  if (args.skip_if_stopped && args.ctl->stop) return;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment (of the shared-window address) for SWIZZLE_128B atoms
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stage_base = smem;                                  // kNSt * kStageBytes
  uint8_t* ai_base = smem + kNSt * kStageBytes;                // 2 * kAIBytes
  uint64_t* bars = reinterpret_cast<uint64_t*>(ai_base + 2 * kAIBytes);
  // barrier slots
  uint64_t* full = bars;                     // [kNSt]
  uint64_t* empty = bars + kNSt;             // [kNSt]
  uint64_t* ai_full = bars + 2 * kNSt;       // [2]
  uint64_t* ai_empty = ai_full + 2;          // [2]
  uint64_t* p_full = ai_full + 4;            // [2]
  uint64_t* p_empty = ai_full + 6;           // [2]
  uint64_t* q_full = ai_full + 8;            // [kMaxC], one per Q column tile
  uint64_t* q_empty = q_full + kMaxC;        // [kMaxC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_empty + kMaxC);
  volatile uint32_t* s_first = tmem_slot + 1;  // strip groups: this CTA is not the item's last arrival

  const int warp = warp_id_uniform();
  const int lane = threadIdx.x & 31;
  const int grp = args.grp > 1 ? args.grp : 1;
  const int half = (int)(blockIdx.x % grp);  // member of the strip group
  const int rng = (int)(blockIdx.x / grp);   // item range index (one per group)
  const int item_b = args.cta_begin[rng];
  const int item_e = args.cta_begin[rng + 1];
  const int nstrips = args.nstrips, nrb = args.nrb, ncb = args.ncb, c = args.c, NR = args.NR, sw = args.sw;
  const int qrot = args.qrot;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNSt; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&ai_full[i]), 1);
      mbar_init(smem_u32(&ai_empty[i]), 1);
      mbar_init(smem_u32(&p_full[i]), 1);
      mbar_init(smem_u32(&p_empty[i]), 4);  // one arrive per epilogue warp
    }
    for (int i = 0; i < kMaxC; ++i) {
      mbar_init(smem_u32(&q_full[i]), 1);
      mbar_init(smem_u32(&q_empty[i]), 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_xh);
    tma_prefetch(&map_xl);
    tma_prefetch(&map_rh);
    tma_prefetch(&map_rl);
    tma_prefetch(&map_ch);
    tma_prefetch(&map_cl);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int item = item_b; item < item_e; ++item) {
        int t, s, rb;
        decode_item(item, nstrips, nrb, t, s, rb);
        int ct, toff;
        k1_half_tiles(s, nstrips, sw, ncb, grp, half, ct, toff);
        const int ab = (item - item_b) & 1;
        const uint32_t ap = ((item - item_b) >> 1) & 1;
        // A^T[:, I] (row operand of Q) for this row block
        mbar_wait(smem_u32(&ai_empty[ab]), ap ^ 1);
        const uint32_t ai = smem_u32(ai_base + ab * kAIBytes);
        const uint32_t aib = smem_u32(&ai_full[ab]);
        mbar_expect_tx(aib, kAIBytes);
        tma_load_2d(ai + 0 * kABox, &map_rh, rb * kTile, 0, aib);
        tma_load_2d(ai + 1 * kABox, &map_rl, rb * kTile, 0, aib);
        tma_load_2d(ai + 2 * kABox, &map_rh, rb * kTile + 64, 0, aib);
        tma_load_2d(ai + 3 * kABox, &map_rl, rb * kTile + 64, 0, aib);
        const int xrow = t * NR + rb * kTile;
        for (int cb = 0; cb < ct; ++cb) {
          const int j0 = (s * sw + toff + cb) * kTile;
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {  // 0: X hi + A_col hi / lo, 1: X lo + A_col hi
            mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
            const uint32_t st = smem_u32(stage_base + stage * kStageBytes);
            const uint32_t fb = smem_u32(&full[stage]);
            const CUtensorMap* mx = sub ? &map_xl : &map_xh;
            mbar_expect_tx(fb, 2 * kXBox + (sub ? 2 : 4) * kABox);
            tma_load_2d(st + 0 * kXBox, mx, j0, xrow, fb);
            tma_load_2d(st + 1 * kXBox, mx, j0 + 64, xrow, fb);
            tma_load_2d(st + kStageX + 0 * kABox, &map_ch, j0, 0, fb);
            tma_load_2d(st + kStageX + 2 * kABox, &map_ch, j0 + 64, 0, fb);
            if (!sub) {
              tma_load_2d(st + kStageX + 1 * kABox, &map_cl, j0, 0, fb);
              tma_load_2d(st + kStageX + 3 * kABox, &map_cl, j0 + 64, 0, fb);
            }
            if (++stage == kNSt) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    // the whole warp walks the schedule (warp-uniform); one elected lane
    // issues each k-step's MMAs and the commits
    {
      const uint32_t id_p = idesc_bf16(K, 0);  // A = X tile, K-major (K-dim = j)
      const uint32_t id_q = idesc_bf16(K, 1);  // A = X tile, MN-major (M = j, K-dim = i)
      const uint32_t id_p2 = idesc_bf16(2 * K, 0);  // merged [hi ; lo] B operand
      const uint32_t id_q2 = idesc_bf16(2 * K, 1);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t owed = 0;     // Q tiles committed for a drain, not yet waited free
      uint32_t qe_par = 0;   // per-tile q_empty parity
      uint32_t restart = 0;  // Q tiles whose next MMA starts a fresh TMEM sum
      for (int item = item_b; item < item_e; ++item) {
        int t, s, rb;
        decode_item(item, nstrips, nrb, t, s, rb);
        int ct, toff;
        k1_half_tiles(s, nstrips, sw, ncb, grp, half, ct, toff);
        const int ts = item / nrb;
        if (item == item_b || (item - 1) / nrb != ts) restart = ~0u;  // a new (t, strip) run
        const bool run_end = item == item_e - 1 || (item + 1) / nrb != ts;
        const int dcb = k1_rot_tile(rb, qrot, c);  // the Q tile drained after this item
        const int idx = item - item_b;
        const int ab = idx & 1;
        const uint32_t ap = (idx >> 1) & 1;
        // (P double-buffered across items. Splitting an item's P over both
        // buffers halves P's TMEM error but made the factors LESS accurate:
        // P's and Q's truncation biases then differ -- the MU update absorbs
        // a common scale, not a P / Q imbalance; profiles/r02_q_rotation.md)
        const int pb = idx & 1;
        const uint32_t pp = (idx >> 1) & 1;
        mbar_wait(smem_u32(&ai_full[ab]), ap);
        mbar_wait(smem_u32(&p_empty[pb]), pp ^ 1);
        tc_fence_after();
        const uint32_t ai = smem_u32(ai_base + ab * kAIBytes);
        const uint32_t p_tmem = tmem + (uint32_t)(c * kQW + pb * kPW);
        for (int cb = 0; cb < ct; ++cb) {
          const uint32_t q_tmem = tmem + (uint32_t)(cb * kQW);
          const uint32_t bit = 1u << cb;
          if (owed & bit) {  // its last drain has read the TMEM tile
            mbar_wait(smem_u32(&q_empty[cb]), (qe_par >> cb) & 1);
            qe_par ^= bit;
            owed &= ~bit;
            tc_fence_after();
          }
          const bool q_fresh = (restart & bit) != 0;
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {  // 0: the X hi plane's products, 1: the X lo plane's
            mbar_wait(smem_u32(&full[stage]), phase);
            tc_fence_after();
            const uint32_t st = smem_u32(stage_base + stage * kStageBytes);
            const uint32_t aj = st + kStageX;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const uint32_t xoff = (ks >> 2) * kXBox + (ks & 3) * 32;
              const uint32_t hoff = (ks >> 2) * 2 * kABox + (ks & 3) * 32;
              const uint32_t loff = hoff + kABox;
              const uint64_t dx = umma_desc(st + xoff, 16, 1024);
              const uint64_t dah = umma_desc(aj + hoff, 16, 1024);
              const uint64_t qx = umma_desc(st + ks * 16 * 128, kXBox, 1024);
              const uint64_t qah = umma_desc(ai + hoff, 16, 1024);
              if (elect_one()) {
                if (sub == 0) {
                  const uint32_t accp = (cb > 0 || ks > 0) ? 1u : 0u;
                  const uint32_t accq = (q_fresh && ks == 0) ? 0u : 1u;
                  if (kMergeP) {
                    tc_mma(p_tmem, dx, dah, id_p2, accp);  // [Xh Ah | Xh Al]
                  } else {
                    tc_mma(p_tmem, dx, dah, id_p, accp);
                    tc_mma(p_tmem, dx, umma_desc(aj + loff, 16, 1024), id_p, 1u);
                  }
                  if (kMergeQ) {
                    tc_mma(q_tmem, qx, qah, id_q2, accq);
                  } else {
                    tc_mma(q_tmem, qx, qah, id_q, accq);
                    tc_mma(q_tmem, qx, umma_desc(ai + loff, 16, 1024), id_q, 1u);
                  }
                } else {
                  tc_mma(p_tmem, dx, dah, id_p, 1u);  // Xl Ah into P's first half
                  tc_mma(q_tmem, qx, qah, id_q, 1u);  // Xl^T Ah_I
                }
              }
              __syncwarp();
            }
            if (elect_one()) tc_commit(smem_u32(&empty[stage]));
            __syncwarp();
            if (++stage == kNSt) {
              stage = 0;
              phase ^= 1;
            }
          }
          restart &= ~bit;
          if (run_end || cb == dcb) {  // tile cb's sum is drained after this item
            if (elect_one()) tc_commit(smem_u32(&q_full[cb]));
            __syncwarp();
            owed |= bit;
            restart |= bit;
          }
        }
        if (elect_one()) {
          tc_commit(smem_u32(&p_full[pb]));
          tc_commit(smem_u32(&ai_empty[ab]));
        }
        __syncwarp();
      }
    }
  } else {
    // ============================ epilogue ================================
    const int quad = warp & 3;                 // TMEM lane quadrant
    const int row = quad * 32 + lane;          // row within the 128-row tile
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    uint32_t qf_par = 0;     // per-tile q_full parity
    uint32_t stored = 0;     // tiles of the current slot written at least once
    int slot = args.cta_slot[blockIdx.x] - 1;
    int slot_ts = -1;        // the (t, strip) the current slot belongs to
    uint64_t pol_keep, pol_norm;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_norm));
    for (int item = item_b; item < item_e; ++item) {
      int t, s, rb;
      decode_item(item, nstrips, nrb, t, s, rb);
      int ct, toff;
      k1_half_tiles(s, nstrips, sw, ncb, grp, half, ct, toff);
      const int ts = item / nrb;
      const bool run_end = item == item_e - 1 || (item + 1) / nrb != ts;
      const int dcb = k1_rot_tile(rb, qrot, c);
      const int idx = item - item_b;
      if (ts != slot_ts) {  // one slot per (CTA, (t, strip) run)
        ++slot;
        slot_ts = ts;
        stored = 0;
      }
      float4* qslot = reinterpret_cast<float4*>(args.Qpart + (size_t)slot * c * kTile * K) + row;
      if (!kRot) stored = 0;  // (lets the compiler drop the read-back path)
      if (item == item_e - 1 && stored != 0) {
        // the CTA's final drain never reads back (a load round trip per tile
        // would sit on the kernel's tail): it stores into a slot of its own;
        // the tiles the old slot never received are zeroed
        for (int cb = 0; cb < ct; ++cb)
          if (!((stored >> cb) & 1)) {
#pragma unroll
            for (int h = 0; h < K / 4; ++h) qslot[((size_t)cb * K / 4 + h) * kTile] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        ++slot;
        stored = 0;
        qslot += (size_t)c * kTile * K / 4;
      }
      // a slot tile a later drain reads back is stored evict-last (an L2
      // set-aside holds it against the X stream); the run's last store releases it
      const uint64_t pol = run_end ? pol_norm : pol_keep;
      if (run_end) {
        // every Q tile of the run: tiles in pairs, each with its own register
        // set, so a read-back load has two tiles of time to land
        float4 o[2][K / 4];
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (u < ct && ((stored >> u) & 1)) {
#pragma unroll
            for (int h = 0; h < K / 4; ++h) o[u][h] = qslot[((size_t)u * K / 4 + h) * kTile];
          }
        for (int cp = 0; cp < ct; cp += 2) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int cb = cp + u;
            if (cb < ct) {
              const bool add = (stored >> cb) & 1;
              k1_drain_q<K, kMergeQ>(tmem + lane_base + (uint32_t)(cb * kQW), smem_u32(&q_full[cb]),
                                     (qf_par >> cb) & 1, smem_u32(&q_empty[cb]), lane,
                                     qslot + (size_t)cb * kTile * K / 4, o[u], add, pol);
              qf_par ^= 1u << cb;
              if (cb + 2 < ct && ((stored >> (cb + 2)) & 1)) {
#pragma unroll
                for (int h = 0; h < K / 4; ++h) o[u][h] = qslot[((size_t)(cb + 2) * K / 4 + h) * kTile];
              }
            }
          }
        }
        stored = 0;  // the next item starts a new run (or the CTA is done)
      } else if (kRot && dcb >= 0 && dcb < ct) {
        // the one tile this item rotates out; its MMAs for the next item wait
        // ~c - 1 tiles later, so this never stalls the tensor pipe
        const bool add = (stored >> dcb) & 1;
        float4 o[K / 4];
        float4* qd = qslot + (size_t)dcb * kTile * K / 4;
        if (add) {
#pragma unroll
          for (int h = 0; h < K / 4; ++h) o[h] = qd[h * kTile];
        }
        k1_drain_q<K, kMergeQ>(tmem + lane_base + (uint32_t)(dcb * kQW), smem_u32(&q_full[dcb]),
                               (qf_par >> dcb) & 1, smem_u32(&q_empty[dcb]), lane, qd, o, add, pol);
        qf_par ^= 1u << dcb;
        stored |= 1u << dcb;
      }
      const int pb = idx & 1;
      const uint32_t pp = (idx >> 1) & 1;
      mbar_wait(smem_u32(&p_full[pb]), pp);
      tc_fence_after();
      float v[K];
#pragma unroll
      for (int h = 0; h < K / 16; ++h)
        tmem_ld16(tmem + lane_base + (uint32_t)(c * kQW + pb * kPW + 16 * h), v + 16 * h);
      if (kMergeP) {
        float v2[K];
#pragma unroll
        for (int h = 0; h < K / 16; ++h)
          tmem_ld16(tmem + lane_base + (uint32_t)(c * kQW + pb * kPW + K + 16 * h), v2 + 16 * h);
#pragma unroll
        for (int d = 0; d < K; ++d) v[d] += v2[d];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&p_empty[pb]));
      if (ct == 0) {  // a group member without tiles in a ragged last strip: no MMA wrote P
#pragma unroll
        for (int d = 0; d < K; ++d) v[d] = 0.f;
      }
      // partial layout [strip][t][row block][K/4][128 rows] float4 (coalesced)
      float4* dst = reinterpret_cast<float4*>(
                        args.Ppart + ((((size_t)s * args.M + t) * NR) + (size_t)rb * kTile) * K) + row;
      if (grp > 1) {
        // Strip groups: the grp CTAs of a group produce P tiles for the same
        // (t, strip, rb). The last to arrive (ticket per buffer slot) sums
        // all of them in member order (deterministic) and writes the strip's
        // one partial; the others store their tile in the group's L2 scratch
        // and move on, so the members never run in lockstep.
        const int b = idx % kPairSlots;
        const unsigned k = (unsigned)(idx / kPairSlots);  // earlier uses of slot b
        unsigned* tk = args.pflag + (size_t)rng * kPairWords;  // [tickets][ready][done][exit]
        unsigned* ready = tk + kPairSlots;
        unsigned* done = ready + kPairSlots;
        float* scr0 = args.Pscr + ((size_t)rng * kPairSlots + b) * grp * kTile * K;  // member tiles
        if (threadIdx.x == 64) {
          // slot b's previous use must be complete (all arrivals and the
          // read) before its ticket is taken: the ticket then counts this
          // item's arrivals even when a member runs kPairSlots items ahead
          // (waits only then)
          if (k > 0)
            while (ld_acquire_u32(done + b) < k) {
            }
          *s_first = (atomicAdd(tk + b, 1u) % (unsigned)grp) != (unsigned)(grp - 1) ? 1u : 0u;
        }
        epi_bar();
        if (*s_first) {
          // evict-last: the tile must survive the X stream until it is read
          // (and discarded)
          uint64_t pol;
          asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
          float4* scr = reinterpret_cast<float4*>(scr0 + (size_t)half * kTile * K) + row;
#pragma unroll
          for (int h = 0; h < K / 4; ++h)
            asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(scr + h * kTile),
                         "f"(v[4 * h]), "f"(v[4 * h + 1]), "f"(v[4 * h + 2]), "f"(v[4 * h + 3]), "l"(pol)
                         : "memory");
          __threadfence();
          epi_bar();
          if (threadIdx.x == 64) red_release_add_u32(ready + b, 1u);
        } else {
          if (threadIdx.x == 64)
            while (ld_acquire_u32(ready + b) < (k + 1) * (unsigned)(grp - 1)) {
            }
          epi_bar();
          float acc[K];
#pragma unroll
          for (int d = 0; d < K; ++d) acc[d] = 0.f;
          for (int qq = 0; qq < grp; ++qq) {  // member order: the same sum whoever arrives last
            if (qq == half) {
#pragma unroll
              for (int d = 0; d < K; ++d) acc[d] += v[d];
            } else {
              const float4* scr = reinterpret_cast<const float4*>(scr0 + (size_t)qq * kTile * K) + row;
#pragma unroll
              for (int h = 0; h < K / 4; ++h) {
                const float4 o = __ldcg(scr + h * kTile);
                acc[4 * h] += o.x;
                acc[4 * h + 1] += o.y;
                acc[4 * h + 2] += o.z;
                acc[4 * h + 3] += o.w;
              }
            }
          }
          epi_bar();  // every row read
          // the tiles are dead: drop their L2 lines without a write-back
          // (else the partial traffic the group saves reappears as scratch
          // write-backs); one 128 B line per thread and member tile
          for (int qq = 0; qq < grp; ++qq) {
            if (qq == half) continue;
            if (threadIdx.x - 64 < K * kTile * 4 / 128) {
              const char* line = reinterpret_cast<const char*>(scr0 + (size_t)qq * kTile * K) +
                                 (size_t)(threadIdx.x - 64) * 128;
              asm volatile("discard.global.L2 [%0], 128;" ::"l"(line) : "memory");
            }
          }
          __threadfence();
          epi_bar();
          if (threadIdx.x == 64) st_release_u32(done + b, k + 1);
#pragma unroll
          for (int h = 0; h < K / 4; ++h)
            dst[h * kTile] = make_float4(acc[4 * h], acc[4 * h + 1], acc[4 * h + 2], acc[4 * h + 3]);
        }
      } else {
#pragma unroll
        for (int h = 0; h < K / 4; ++h)
          dst[h * kTile] = make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
      }
    }
    // the group's counters start from zero in the next launch: the last
    // member to finish resets them (all are done with them by then)
    if (grp > 1 && threadIdx.x == 64) {
      unsigned* f = args.pflag + (size_t)rng * kPairWords;
      __threadfence();
      if (atomicAdd(f + 3 * kPairSlots, 1u) == (unsigned)(grp - 1)) {
        for (int w = 0; w < kPairWords; ++w) f[w] = 0u;
        __threadfence();
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

template <int K>
constexpr uint32_t k1_smem_bytes() {  // same for both MQ variants
  return 1024 /*align slack*/ + K1Stages<K>::kNSt * K1Stages<K>::kSubBytes + 2 * (4 * K * 128) +
         (2 * K1Stages<K>::kNSt + 8 + 2 * kMaxC) * 8 + 16;
}

// Deterministic reduction of the partials:
//   P[t][i] = sum_s Ppart[t][s][i]                         (i < NR)
//   Q[t][j] = sum_{slots of (t, strip(j))} Qpart[slot][j - strip0]   (j < NC)
// Body over a grid-stride range (thread g0 of gstride); also run as phase 1
// of the fused k-wide chain (k2_chain.cuh).
// One float4 of P (row i of slice t, columns 4 q4 .. 4 q4 + 3): strips summed in order.
RK_DEV void k1_reduce_p4(const float* __restrict__ Ppart, float* __restrict__ P, int NR, int K, int M,
                         int nstrips, int t, int i, int q4) {
  // loads batched 4 at a time (independent, in flight together), sums kept in strip order
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const size_t sstride = (size_t)M * NR * K / 4;  // float4s between strips
  const float4* src = reinterpret_cast<const float4*>(Ppart + (((size_t)t * NR) + (i & ~(kTile - 1))) * K) +
                      q4 * kTile + (i & (kTile - 1));
  int s = 0;
  for (; s + 4 <= nstrips; s += 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = src[(size_t)(s + u) * sstride];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
    }
  }
  for (; s < nstrips; ++s) {
    const float4 v = src[(size_t)s * sstride];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  reinterpret_cast<float4*>(P + ((size_t)t * NR + i) * K)[q4] = acc;
}

// One float4 of Q (row j of slice t): the Q-partial slots of its strip in order.
RK_DEV void k1_reduce_q4(const float* __restrict__ Qpart, const int* __restrict__ slot_first,
                         const int* __restrict__ slot_count, float* __restrict__ Q, int NC, int K, int c,
                         int nstrips, int t, int j, int q4, int sw = 0, int grp = 1) {
  // slots hold c column tiles; a strip has sw tiles (sw = c, or up to grp c
  // split between the CTAs of a group: slots keyed (t, strip, member))
  const int W = c * kTile;
  const int swt = sw ? sw : c;
  grp = grp > 1 ? grp : 1;
  const int s = j / (swt * kTile);
  const int jt = (j - s * swt * kTile) / kTile;  // tile within the strip
  int half = 0, toff = 0;
  for (int q = 1; q < grp; ++q) {  // the member whose tiles hold jt
    int ctq, tq;
    k1_half_tiles(s, nstrips, swt, NC / kTile, grp, q, ctq, tq);
    if (jt >= tq) {
      half = q;
      toff = tq;
    }
  }
  const int jl = (jt - toff) * kTile + (j & (kTile - 1));  // column within the slot
  const int key = (t * nstrips + s) * grp + half;
  const int f = slot_first[key], nsl = slot_count[key];
  float4 qa = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* src = reinterpret_cast<const float4*>(Qpart + ((size_t)f * W + (jl & ~(kTile - 1))) * K) +
                      q4 * kTile + (jl & (kTile - 1));
  const size_t qstride = (size_t)W * K / 4;  // float4s between slots
  int q = 0;
  for (; q + 4 <= nsl; q += 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = src[(size_t)(q + u) * qstride];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      qa.x += v[u].x; qa.y += v[u].y; qa.z += v[u].z; qa.w += v[u].w;
    }
  }
  for (; q < nsl; ++q) {
    const float4 v = src[(size_t)q * qstride];
    qa.x += v.x; qa.y += v.y; qa.z += v.z; qa.w += v.w;
  }
  reinterpret_cast<float4*>(Q + ((size_t)t * NC + j) * K)[q4] = qa;
}

RK_DEV void k1_reduce_body(const float* __restrict__ Ppart, const float* __restrict__ Qpart,
                           const int* __restrict__ slot_first, const int* __restrict__ slot_count,
                           float* __restrict__ P, float* __restrict__ Q, int NR, int NC, int K, int M, int c,
                           int nstrips, int64_t g0, int64_t gstride, int sw = 0, int grp = 1) {
  const int K4 = K / 4;
  const int64_t totalP = (int64_t)M * NR * K4;
  const int64_t total = totalP + (int64_t)M * NC * K4;
#pragma unroll 2
  for (int64_t e = g0; e < total; e += gstride) {
    // consecutive threads take consecutive rows of one float4 column: the
    // partials' [row block][K/4][128] layout makes their loads contiguous
    if (e < totalP) {
      const int r = (int)(e % kTile);
      const int64_t rest = e / kTile;
      const int q4 = (int)(rest % K4);
      const int64_t ti = (rest / K4) * kTile + r;
      k1_reduce_p4(Ppart, P, NR, K, M, nstrips, (int)(ti / NR), (int)(ti % NR), q4);
    } else {
      const int64_t e2 = e - totalP;
      const int r = (int)(e2 % kTile);
      const int64_t rest = e2 / kTile;
      const int q4 = (int)(rest % K4);
      const int64_t tj = (rest / K4) * kTile + r;
      k1_reduce_q4(Qpart, slot_first, slot_count, Q, NC, K, c, nstrips, (int)(tj / NC), (int)(tj % NC), q4, sw,
                   grp);
    }
  }
}

__global__ void __launch_bounds__(256) k1_reduce(const Ctl* __restrict__ ctl,
                                                 const float* __restrict__ Ppart,
                                                 const float* __restrict__ Qpart,
                                                 const int* __restrict__ slot_first,
                                                 const int* __restrict__ slot_count,
                                                 float* __restrict__ P, float* __restrict__ Q,
                                                 int NR, int NC, int K, int M, int c, int nstrips,
                                                 int skip_if_stopped, int sw, int grp) {
  pdl_entry();
  if (skip_if_stopped && ctl->stop) return;
  k1_reduce_body(Ppart, Qpart, slot_first, slot_count, P, Q, NR, NC, K, M, c, nstrips,
                 (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x, sw, grp);
}

}  // namespace tc
}  // namespace rk
