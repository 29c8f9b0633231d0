// rescal_b200.cu — C-ABI implementation (include/rescal_b200.h).
//
// One handle = one GPU, one CUDA stream, all tensor/factor buffers resident
// in HBM. An MU iteration (rescal.py:114-146 + the trace of :215-224) is the
// kernel sequence
//   K1  slice contraction  P_t = X_t A_col, Q_t = X_t^T A_row   (tcgen05 or SIMT)
//   K5  direct residual of the current iterate (only in the small-error regime)
//   K2a G / S_t partials   K2f per-slice core update + M_t   K2m trace/commit
//   K2b A update + next-iteration operand planes
// captured once into a CUDA graph and replayed; stop conditions live in a
// device control block so queued iterations become no-ops without host syncs.
// On a p_r x p_c grid the same kernels run on the local block with NCCL
// all-gather / all-reduce / reduce-scatter in between.

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/rescal_b200.h"
#include "k1_tc.cuh"
#include <nvtx3/nvToolsExt.h>
#include "peer.cuh"
#include "rk_kernels.cuh"
#include "sparse.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

using rk::Ctl;

namespace {

thread_local std::string g_err;

struct RkError {
  int code;
  std::string msg;
};

#define RK_CUDA(expr)                                                                      \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      throw RkError{RK_ERR_DEVICE, std::string(#expr) + ": " + cudaGetErrorString(_e)};    \
  } while (0)

#define RK_NCCL(expr)                                                                      \
  do {                                                                                     \
    ncclResult_t _r = (expr);                                                              \
    if (_r != ncclSuccess)                                                                 \
      throw RkError{RK_ERR_GRID, std::string(#expr) + ": " + ncclGetErrorString(_r)};      \
  } while (0)

#define RK_REQUIRE(cond, code, msg)             \
  do {                                          \
    if (!(cond)) throw RkError{(code), (msg)}; \
  } while (0)

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return RK_OK;
  } catch (const RkError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RK_ERR_DEVICE;
  }
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// Process-wide device-memory cache (as PyTorch's caching allocator): freed
// blocks are kept per (device, size class) and reused by later handles
// (repeated rescal_solve / RESCALk members / tests), so handle teardown does
// not pay cudaFree's unmapping and creation does not pay cudaMalloc's
// mapping of tens of GB. Blocks are released on an allocation failure (then
// the allocation is retried) or by rk_release_cached_memory().
struct DevPool {
  std::mutex mu;
  std::unordered_map<void*, std::pair<int, size_t>> live;  // ptr -> (device, bytes)
  std::multimap<std::pair<int, size_t>, void*> idle;        // (device, bytes) -> ptr
  // guard mode (rk_debug_guards; compute-sanitizer is not available on the
  // GPU pool): every new block is followed by kGuard bytes of a fixed
  // pattern, checked on free and by rk_debug_check_guards
  bool guard = false;
  std::unordered_map<void*, size_t> guarded;  // ptr -> requested bytes (guard starts there)
  int64_t violations = 0;
};
constexpr size_t kGuard = 64 << 10;
constexpr unsigned char kGuardByte = 0xA5;

DevPool& dev_pool() {
  static DevPool* p = new DevPool();  // process lifetime (no teardown-order hazards)
  return *p;
}

size_t pool_class(size_t b) {
  return b >= (1u << 20) ? (size_t)round_up((int64_t)b, 2 << 20) : (size_t)round_up((int64_t)b, 512);
}

void pool_release(int dev) {
  DevPool& P = dev_pool();
  std::lock_guard<std::mutex> lk(P.mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto it = P.idle.begin(); it != P.idle.end();) {
    if (dev < 0 || it->first.first == dev) {
      cudaSetDevice(it->first.first);
      cudaFree(it->second);
      it = P.idle.erase(it);
    } else {
      ++it;
    }
  }
  cudaSetDevice(cur);
}

// bytes of the guard band of block p that lost the pattern (caller holds mu)
int64_t guard_damage(void* p, size_t req, int dev) {
  std::vector<unsigned char> g(kGuard);
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(dev);
  cudaDeviceSynchronize();
  cudaMemcpy(g.data(), static_cast<unsigned char*>(p) + req, kGuard, cudaMemcpyDeviceToHost);
  cudaSetDevice(cur);
  int64_t bad = 0;
  for (unsigned char c : g) bad += c != kGuardByte;
  return bad;
}

void* pool_alloc(size_t bytes) {
  DevPool& P = dev_pool();
  int dev = 0;
  RK_CUDA(cudaGetDevice(&dev));
  const size_t b = pool_class(bytes);
  if (P.guard) {  // no reuse: a fresh block with the guard band right after the request
    void* p = nullptr;
    RK_CUDA(cudaMalloc(&p, bytes + kGuard));
    RK_CUDA(cudaMemset(static_cast<unsigned char*>(p) + bytes, kGuardByte, kGuard));
    std::lock_guard<std::mutex> lk(P.mu);
    P.live[p] = {dev, bytes};
    P.guarded[p] = bytes;
    return p;
  }
  {
    std::lock_guard<std::mutex> lk(P.mu);
    // best fit within 12.5 % of the request
    auto it = P.idle.lower_bound({dev, b});
    if (it != P.idle.end() && it->first.first == dev && it->first.second <= b + b / 8) {
      void* p = it->second;
      P.live[p] = it->first;
      P.idle.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, b);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    pool_release(dev);
    e = cudaMalloc(&p, b);
  }
  if (e != cudaSuccess) throw RkError{RK_ERR_DEVICE, std::string("cudaMalloc: ") + cudaGetErrorString(e)};
  std::lock_guard<std::mutex> lk(P.mu);
  P.live[p] = {dev, b};
  return p;
}

template <typename T>
T* dalloc(size_t count) {
  if (count == 0) count = 1;
  void* p = pool_alloc(count * sizeof(T));
  RK_CUDA(cudaMemset(p, 0, count * sizeof(T)));
  // the engine stream is non-blocking w.r.t. the legacy stream the memset
  // ran on: finish the zeroing (and any earlier user of a reused block)
  // before an engine kernel can touch the buffer
  RK_CUDA(cudaDeviceSynchronize());
  return static_cast<T*>(p);
}

void dfree(void* p) {
  if (!p) return;
  DevPool& P = dev_pool();
  std::lock_guard<std::mutex> lk(P.mu);
  auto it = P.live.find(p);
  if (it == P.live.end()) {  // not from dalloc
    cudaFree(p);
    return;
  }
  auto g = P.guarded.find(p);
  if (g != P.guarded.end()) {  // guard mode: check the band, give the block back to the driver
    P.violations += guard_damage(p, g->second, it->second.first);
    P.guarded.erase(g);
    P.live.erase(it);
    cudaFree(p);
    return;
  }
  P.idle.insert({it->second, p});
  P.live.erase(it);
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    RK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    RK_REQUIRE(q == cudaDriverEntryPointSuccess && p, RK_ERR_DEVICE,
               "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// bf16 row-major matrix [rows][cols], box {64 cols, box_rows}, 128B swizzle
CUtensorMap make_map(const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  RK_REQUIRE(r == CUDA_SUCCESS, RK_ERR_DEVICE, "cuTensorMapEncodeTiled failed");
  return m;
}

}  // namespace

struct rk_handle {
  int dev = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  // problem
  int64_t n = 0, m = 0;  // global n, slices
  int k = 0, K = 0;      // rank, padded rank
  int engine = RK_ENGINE_AUTO;
  int requested_engine = RK_ENGINE_AUTO;
  // local block (NR x NC padded; rows_valid x cols_valid real)
  int64_t NR = 0, NC = 0, rows_valid = 0, cols_valid = 0;
  // grid
  int pr = 1, pc = 1, rank = 0, gi = 0, gj = 0;
  int64_t piece = 0;  // b = ceil(n / p)
  ncclComm_t world = nullptr, rowc = nullptr, colc = nullptr;
  std::vector<int64_t> colmap;  // local col -> global col
  int64_t* d_colmap = nullptr;
  // tensor
  __nv_bfloat16 *Xh = nullptr, *Xl = nullptr, *Xh0 = nullptr, *Xl0 = nullptr;
  bool have_x = false, perturbed = false;
  double norm2 = 0.0, norm2_dev = 0.0, norm2_dev0 = 0.0, norm2_orig = 0.0;
  // factors and working copies
  double *Arow = nullptr, *Acol = nullptr;  // alias on one GPU
  float *A32row = nullptr, *A32col = nullptr;
  __nv_bfloat16 *ATh_row = nullptr, *ATl_row = nullptr, *ATh_col = nullptr, *ATl_col = nullptr;
  double *R = nullptr, *Rnext = nullptr, *Mt = nullptr, *Mm = nullptr, *tt = nullptr;
  double* part = nullptr;   // K2a partials [M+1][nchunks][K^2]
  double* red = nullptr;    // reduced G, S_t (+ residual scalar): the grid all-reduce buffer
  int nb = 1;               // K2a row chunks
  int chunk_rows = 64;
  unsigned* counters = nullptr;  // last-block tickets (self-resetting)
  bool skip_comm = false;        // experiments only: skip the per-iteration NCCL calls
  bool fast = false;             // single GPU, K in {16, 32}: k2a_v4 / k2b_v4 path
  float* W32 = nullptr;          // [M][2][K][K] fp32 (R_t^T ; R_t) for k2b_v4
  int *d_simt_first = nullptr, *d_simt_count = nullptr;
  double* gscratch = nullptr;
  double *UI = nullptr, *UJ = nullptr;  // grid numerator partials
  double *regS = nullptr, *regG = nullptr, *regT = nullptr, *regRn = nullptr;
  int* d_iters = nullptr;
  float *P = nullptr, *Q = nullptr;
  double* rpart = nullptr;
  int nr = 1;
  double* trace_dev = nullptr;
  int trace_cap = 0;
  Ctl* ctl = nullptr;
  Ctl* ctl_host = nullptr;   // pinned
  int* stop_host = nullptr;  // pinned [2]
  double* npart = nullptr;   // upload norm partials
  double* npart2 = nullptr;
  int nnp = 0;
  // tcgen05 schedule
  int c = 0, nstrips = 0, grid_tc = 0, nslots = 0, qrot = 1;
  int sw = 0;           // K1 column tiles per strip (c, or up to grp c with strip groups)
  int k1_grp = 1;       // K1 CTAs per strip group (1, 2, 4)
  float* Pscr = nullptr;      // strip groups: the members' P tiles
  unsigned* pflag = nullptr;  // strip groups: ticket / ready / done / exit counters
  bool k1_mq = true;  // K1 merges the Q hi/lo operands (always at K = 16; see k1_merge_q)
  size_t smem_tc = 0;
  float *Ppart = nullptr, *Qpart = nullptr;
  int *d_cta_begin = nullptr, *d_cta_slot = nullptr, *d_slot_first = nullptr,
      *d_slot_count = nullptr;
  CUtensorMap maps[6];
  // graph
  // [track][batched]: one iteration, or kGraphBatch iterations in one graph;
  // the untracked variants leave out the (then always gated-off) K5 node
  cudaGraphExec_t graphs[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  int graph_launches[2][2] = {{0, 0}, {0, 0}};
  bool use_graph = true;
  // timing
  bool profile = false;
  cudaEvent_t ev_run0 = nullptr, ev_run1 = nullptr;
  std::vector<cudaEvent_t> ev_k1;
  // per-phase timing (profile mode): events at phase boundaries of each iteration
  static constexpr int kPhases = 6;
  std::vector<cudaEvent_t> ev_ph;
  int ph_iters = 0;
  double ph_ms[kPhases] = {0, 0, 0, 0, 0, 0};
  double last_ms = 0.0, k1_ms_sum = 0.0;
  int k1_count = 0, launches = 0;
  static constexpr int kGraphBatch = 16;
  double eps = 1e-16;

  // sparse tensor (CSR + device-built CSC, fp32 values)
  bool sparse = false;
  int64_t nnz = 0;
  int64_t *csr_ptr = nullptr, *csc_ptr = nullptr;
  int *csr_idx = nullptr, *csc_idx = nullptr;
  float *csr_val = nullptr, *csc_val = nullptr, *csr_val0 = nullptr, *csc_val0 = nullptr;
  double* numer = nullptr;  // [n][K] A numerator (sparse path, grid)
  double* gpart = nullptr;  // sp_gram chunk partials [(M+1)][nchunk][K*K]
  float4* wfrag = nullptr;  // per-lane TF32 hi/lo B fragments of [R_t^T ; R_t] (sparse, K = 16)
  int gchunks = 0;

  // peer-memory grid exchange (peer.cuh): IPC arena of every rank, epochs
  bool peer = false;
  bool peer_tried = false;
  char* arena = nullptr;
  std::vector<void*> peer_open;  // mapped peer arenas (closed on teardown)
  unsigned* pep = nullptr;       // epochs + tickets [8]
  rk::peer::Args pargs{};
  int64_t peer_key[4] = {0, 0, 0, 0};

  bool grid() const { return pr * pc > 1; }
};

namespace {

void drop_graphs(rk_handle* h) {
  for (auto& row : h->graphs)
    for (auto& g : row)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
}

// Dense K in {16, 32} (one GPU or a grid rank): G and S_t on tensor cores
// (sparse.cuh sp_gram_tc_k, TF32 3-pass, fp64 per 32 rows) over the reduced
// P instead of the SIMT cluster kernel k2a_v4 (cfg2 K2a 27 -> 16 us, cfg3
// 197 -> 110 us).
bool k1_tc_k(int K);
bool dense_gram_tc(const rk_handle* h) { return !h->sparse && k1_tc_k(h->K); }

size_t k2f_smem(int K) {
  size_t s = (size_t)5 * K * (K + 1) * sizeof(double);  // row stride K + 1 (mm_kk_t)
  return s <= 200 * 1024 ? s : 0;
}

void free_factor_buffers(rk_handle* h) {
  drop_graphs(h);
  dfree(h->numer);
  h->numer = nullptr;
  dfree(h->gpart);
  h->gpart = nullptr;
  dfree(h->wfrag);
  h->wfrag = nullptr;
  void* ptrs[] = {h->Arow, h->A32row, h->ATh_row, h->ATl_row, h->R, h->Rnext, h->Mt, h->Mm, h->tt,
                  h->part, h->red, h->gscratch, h->counters, h->W32, h->d_simt_first,
                  h->d_simt_count, h->UI, h->UJ, h->regS, h->regG, h->regT,
                  h->regRn, h->P, h->Q, h->rpart, h->Ppart, h->Qpart, h->d_cta_begin,
                  h->d_cta_slot, h->d_slot_first, h->d_slot_count, h->Pscr, h->pflag};
  for (void* p : ptrs) dfree(p);
  h->Pscr = nullptr;
  h->pflag = nullptr;
  if (h->Acol != h->Arow) dfree(h->Acol);
  if (h->A32col != h->A32row) dfree(h->A32col);
  if (h->ATh_col != h->ATh_row) dfree(h->ATh_col);
  if (h->ATl_col != h->ATl_row) dfree(h->ATl_col);
  h->Arow = h->Acol = nullptr;
  h->A32row = h->A32col = nullptr;
  h->ATh_row = h->ATl_row = h->ATh_col = h->ATl_col = nullptr;
  h->R = h->Rnext = h->Mt = h->Mm = h->tt = h->part = h->red = h->gscratch = nullptr;
  h->counters = nullptr;
  h->W32 = nullptr;
  h->d_simt_first = h->d_simt_count = nullptr;
  h->UI = h->UJ = h->regS = h->regG = h->regT = h->regRn = nullptr;
  h->P = h->Q = nullptr;
  h->rpart = nullptr;
  h->Ppart = h->Qpart = nullptr;
  h->d_cta_begin = h->d_cta_slot = h->d_slot_first = h->d_slot_count = nullptr;
}

// K = 32: merge Q's hi/lo operands (4 MMAs per k-step instead of 5) only when
// that does not add column strips: merged Q accumulators are 2K wide, so a
// strip holds 6 column tiles instead of 12, and every extra strip is one more
// copy of P written by K1 and read by k1_reduce. At cfg3 (256 column tiles)
// merging measured 79.8 vs 81.2 it/s (same K1 time: the MMA issue is no
// longer the bound once it runs warp-uniform; profiles/r02k1_*.json).
bool k1_merge_q(int K, int64_t NC) {
  if (K == 16) return true;
  if (K > 32) return false;
  const int64_t ncb = NC / 128;
  return (ncb + 5) / 6 == (ncb + 11) / 12;
}

using K1Kernel = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap,
                         rk::tc::K1Args);

K1Kernel k1_kernel_of(const rk_handle* h) {
  using namespace rk::tc;
  if (h->K == 16) return k1_tc_kernel<16, true>;
  if (h->K == 48) return k1_tc_kernel<48, false>;
  if (h->K == 64) return k1_tc_kernel<64, false>;
  return h->k1_mq ? k1_tc_kernel<32, true> : k1_tc_kernel<32, false>;
}

bool k1_tc_k(int K) { return K == 16 || K == 32 || K == 48 || K == 64; }

using K2bKernel = void (*)(rk::Ctl*, double*, float*, __nv_bfloat16*, __nv_bfloat16*, const float*, const float*,
                          const float*, const double*, int, int, int, double);
K2bKernel k2b_v4_of(int K, int rpt) {
  using namespace rk;
  switch (K) {
    case 16: return rpt > 1 ? k2b_v4<16, 2> : k2b_v4<16, 1>;
    case 48: return rpt > 1 ? k2b_v4<48, 3> : k2b_v4<48, 1>;
    case 64: return rpt > 1 ? k2b_v4<64, 4> : k2b_v4<64, 1>;
    default: return rpt > 1 ? k2b_v4<32, 2> : k2b_v4<32, 1>;
  }
}

using SpGramTcKernel = void (*)(const rk::Ctl*, const float*, const float*, int, int, int, int, double*, int,
                                const float*, int);
SpGramTcKernel sp_gram_tc_of(int K) {
  switch (K) {
    case 16: return rk::sp::sp_gram_tc_k<16>;
    case 48: return rk::sp::sp_gram_tc_k<48>;
    case 64: return rk::sp::sp_gram_tc_k<64>;
    default: return rk::sp::sp_gram_tc_k<32>;
  }
}

// TMEM columns of one P buffer / one Q accumulator of K1<K, MQ>
int k1_pw(int K, bool mq) {
  using namespace rk::tc;
  switch (K) {
    case 16: return K1Cfg<16, true>::kPW;
    case 48: return K1Cfg<48, false>::kPW;
    case 64: return K1Cfg<64, false>::kPW;
    default: return mq ? K1Cfg<32, true>::kPW : K1Cfg<32, false>::kPW;
  }
}
int k1_qw(int K, bool mq) {
  using namespace rk::tc;
  switch (K) {
    case 16: return K1Cfg<16, true>::kQW;
    case 48: return K1Cfg<48, false>::kQW;
    case 64: return K1Cfg<64, false>::kQW;
    default: return mq ? K1Cfg<32, true>::kQW : K1Cfg<32, false>::kQW;
  }
}
size_t k1_smem(int K) {
  using namespace rk::tc;
  switch (K) {
    case 16: return k1_smem_bytes<16>();
    case 48: return k1_smem_bytes<48>();
    case 64: return k1_smem_bytes<64>();
    default: return k1_smem_bytes<32>();
  }
}

// K1's rotating Q drains (k1_tc.cuh): one Q tile drained after every p-th
// row block bounds each TMEM sum to p*c row blocks. p = 1 by default: at
// n = 32768, k = 32 Q's relative error drops from 5.7e-5 to 6.2e-6 and the
// cfg3-shape factors after 3 iterations from relR 9.6e-5 (4 % inside the
// 1e-4 tolerance) to 1.4e-6 -- fp32-class, as north_star's "fp32-accurate"
// split precision asks -- for ~1.5 % more K1 time at cfg3 (slot read-backs;
// profiles/r02_q_rotation.md). RK_K1_QROT=0 turns it off (measurement only).
int k1_qrot() {
  const char* e = std::getenv("RK_K1_QROT");
  return e ? std::max(0, std::atoi(e)) : 1;
}

// K1 strip groups: grp CTAs share a strip (k1_tc.cuh). 2 from 8 strips on,
// 4 from 16; RK_K1_GRP=g forces g (1 = off; measurement only).
constexpr int kPairMinStrips = 8;
constexpr int kQuadMinStrips = 16;
int k1_grp_for(int nstrips) {
  const char* e = std::getenv("RK_K1_GRP");
  if (e) {
    const int g = std::atoi(e);
    return g >= 4 ? 4 : g >= 2 ? 2 : 1;
  }
  return nstrips >= kQuadMinStrips ? 4 : nstrips >= kPairMinStrips ? 2 : 1;
}

// Balanced item ranges and Q-partial slots for the tcgen05 K1 (see k1_tc.cuh).
void plan_tc(rk_handle* h) {
  const int K = h->K;
  const int nrb = (int)(h->NR / 128), ncb = (int)(h->NC / 128);
  h->k1_mq = k1_merge_q(K, h->NC);
  const int pw = k1_pw(K, h->k1_mq);
  const int qw = k1_qw(K, h->k1_mq);
  const int cmax = (512 - 2 * pw) / qw;  // TMEM columns: c Q accumulators + 2 P buffers
  const int M = (int)h->m;
  int c = std::min(cmax, ncb);
  // small tensors (cfg1: 2 x 2 tiles per slice) have fewer items than SMs:
  // narrower strips spread the tiles over more CTAs (each CTA's K1 latency is
  // TMEM alloc + one TMA round trip + its MMAs), at the price of a few more
  // (tiny) P partials
  while (c > 1 && (int64_t)M * ((ncb + c - 1) / c) * nrb < h->num_sms) c = (c + 1) / 2;
  int nstrips = (ncb + c - 1) / c;
  c = (ncb + nstrips - 1) / nstrips;
  nstrips = (ncb + c - 1) / c;
  // Strip groups (k1_tc.cuh): from 8 strips on, grp = 2 (from 16: 4) CTAs
  // share a strip of up to grp c tiles and write ONE P partial for it (1/grp
  // of the partial traffic): pairs cut K1 + k1_reduce by 3 % at 10-22 strips;
  // neutral at cfg2's 5 (ncb 64, K 16), which stays ungrouped
  // (profiles/r02_pairs.md).
  const int grp = nstrips >= 2 ? k1_grp_for(nstrips) : 1;
  const bool pair = grp > 1;
  int sw = c;
  if (pair) {
    nstrips = (ncb + grp * cmax - 1) / (grp * cmax);
    sw = (ncb + nstrips - 1) / nstrips;
    nstrips = (ncb + sw - 1) / sw;
    c = (sw + grp - 1) / grp;
  }
  if (c > rk::tc::kMaxC) throw std::runtime_error("K1 strip wider than kMaxC tiles");
  h->c = c;
  h->sw = sw;
  h->k1_grp = grp;
  h->nstrips = nstrips;
  const int64_t n_items = (int64_t)M * nstrips * nrb;
  auto tiles_of = [&](int64_t item, int half) {
    int ct, toff;
    rk::tc::k1_half_tiles((int)((item / nrb) % nstrips), nstrips, sw, ncb, grp, half, ct, toff);
    return ct;
  };
  int64_t total = 0;
  for (int64_t it = 0; it < n_items; ++it) total += tiles_of(it, 0);
  // item ranges: one per CTA, or one per strip group (all members walk it)
  const int ranges = (int)std::min<int64_t>(h->num_sms / grp, n_items);
  const int grid = grp * ranges;
  std::vector<int> begin(ranges + 1, 0);
  int64_t cum = 0, it = 0;
  for (int g = 0; g < ranges; ++g) {
    begin[g] = (int)it;
    const int64_t target = total * (g + 1) / ranges;
    while (it < n_items && cum + tiles_of(it, 0) <= target) cum += tiles_of(it++, 0);
    if (it == begin[g] && it < n_items) cum += tiles_of(it++, 0);  // at least one item
  }
  begin[ranges] = (int)n_items;
  // slots: one per (CTA, (t, strip) run) in item order, plus a fresh one for
  // a CTA's final drain when its last run already stored (mirrors the
  // epilogue's rule in k1_tc.cuh exactly). Keys (t, strip[, half]); with
  // pairs all even CTAs are numbered first, so every key's slots are
  // consecutive (k1_reduce_q4).
  h->qrot = K <= 32 ? k1_qrot() : 0;
  const int halves = grp;
  std::vector<int> cta_slot(grid, 0), slot_first(M * nstrips * halves, 0), slot_count(M * nstrips * halves, 0);
  int slots = 0;
  auto new_slot = [&](int key) {
    if (slot_count[key] == 0) slot_first[key] = slots;
    slot_count[key] += 1;
    ++slots;
  };
  for (int half = 0; half < halves; ++half)
    for (int r = 0; r < ranges; ++r) {
      const int g = grp * r + half;
      cta_slot[g] = slots;
      int slot_ts = -1;
      bool stored = false;
      for (int i = begin[r]; i < begin[r + 1]; ++i) {
        const int ts = i / nrb, rb = i % nrb;
        const int key = ts * halves + half;
        const int ct = tiles_of(i, half);
        const bool run_end = i == begin[r + 1] - 1 || (i + 1) / nrb != ts;
        if (ts != slot_ts) {
          new_slot(key);
          slot_ts = ts;
          stored = false;
        }
        if (i == begin[r + 1] - 1 && stored) new_slot(key);
        if (run_end)
          stored = false;
        else if (rk::tc::k1_rot_tile(rb, h->qrot, c) >= 0 && rk::tc::k1_rot_tile(rb, h->qrot, c) < ct)
          stored = true;
      }
    }
  if (pair) {
    h->Pscr = dalloc<float>((size_t)ranges * rk::tc::kPairSlots * grp * 128 * K);
    h->pflag = dalloc<unsigned>((size_t)ranges * rk::tc::kPairWords);
    RK_CUDA(cudaMemset(h->pflag, 0, sizeof(unsigned) * ranges * rk::tc::kPairWords));
  }
  h->grid_tc = grid;
  h->nslots = slots;
  const int nkeys = M * nstrips * halves;
  h->d_cta_begin = dalloc<int>(ranges + 1);
  h->d_cta_slot = dalloc<int>(grid);
  h->d_slot_first = dalloc<int>(nkeys);
  h->d_slot_count = dalloc<int>(nkeys);
  RK_CUDA(cudaMemcpy(h->d_cta_begin, begin.data(), sizeof(int) * (ranges + 1), cudaMemcpyHostToDevice));
  RK_CUDA(cudaMemcpy(h->d_cta_slot, cta_slot.data(), sizeof(int) * grid, cudaMemcpyHostToDevice));
  RK_CUDA(cudaMemcpy(h->d_slot_first, slot_first.data(), sizeof(int) * nkeys, cudaMemcpyHostToDevice));
  RK_CUDA(cudaMemcpy(h->d_slot_count, slot_count.data(), sizeof(int) * nkeys, cudaMemcpyHostToDevice));
  h->Ppart = dalloc<float>((size_t)M * nstrips * h->NR * K);
  h->Qpart = dalloc<float>((size_t)slots * c * 128 * K);
  // the slots being added into (one per CTA) are stored evict-last; give
  // them an L2 set-aside so the policy holds against the X stream
  if (h->qrot) {
    int dev = 0, maxp = 0;
    RK_CUDA(cudaGetDevice(&dev));
    RK_CUDA(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
    // (sized to the live slots: the device maximum, 83 MB, slows the X
    // stream itself by 10 %, profiles/r02_q_rotation.md)
    // live evict-last lines: one slot of c tiles per CTA, plus the strip
    // groups' scratch tiles; 1.3x of them (cfg3: 48 MB; 36 MB left 0.4 GB
    // of write-backs, 64 MB measured no better)
    const size_t tile = (size_t)128 * K * sizeof(float);
    const size_t live = (size_t)grid * c * tile + (grp > 1 ? (size_t)ranges * rk::tc::kPairSlots * grp * tile : 0);
    const size_t want = std::min<size_t>((size_t)maxp, live * 13 / 10);
    size_t cur = 0;
    RK_CUDA(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
    if (want > cur) RK_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
  }
  h->maps[0] = make_map(h->Xh, h->NC, (uint64_t)M * h->NR, 128);
  h->maps[1] = make_map(h->Xl, h->NC, (uint64_t)M * h->NR, 128);
  h->maps[2] = make_map(h->ATh_row, h->NR, K, K);
  h->maps[3] = make_map(h->ATl_row, h->NR, K, K);
  h->maps[4] = make_map(h->ATh_col, h->NC, K, K);
  h->maps[5] = make_map(h->ATl_col, h->NC, K, K);
  h->smem_tc = k1_smem(K);
  RK_CUDA(cudaFuncSetAttribute(k1_kernel_of(h), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->smem_tc));
}

void alloc_factor_buffers(rk_handle* h) {
  const int K = h->K;
  const int64_t M = h->m;
  const size_t KK = (size_t)K * K;
  h->Arow = dalloc<double>((size_t)h->NR * K);
  h->A32row = dalloc<float>((size_t)h->NR * K);
  h->ATh_row = dalloc<__nv_bfloat16>((size_t)h->NR * K);
  h->ATl_row = dalloc<__nv_bfloat16>((size_t)h->NR * K);
  if (h->grid()) {
    h->Acol = dalloc<double>((size_t)h->NC * K);
    h->A32col = dalloc<float>((size_t)h->NC * K);
    h->ATh_col = dalloc<__nv_bfloat16>((size_t)h->NC * K);
    h->ATl_col = dalloc<__nv_bfloat16>((size_t)h->NC * K);
    h->UI = dalloc<double>((size_t)h->NR * K);
    h->UJ = dalloc<double>((size_t)h->NC * K);
  } else {
    h->Acol = h->Arow;
    h->A32col = h->A32row;
    h->ATh_col = h->ATh_row;
    h->ATl_col = h->ATl_row;
  }
  h->R = dalloc<double>(M * KK);
  h->Rnext = dalloc<double>(M * KK);
  h->Mt = dalloc<double>(M * KK);
  h->Mm = dalloc<double>(KK);
  h->tt = dalloc<double>(2 * M);
  // K2a row chunks: <= 128 chunks of >= 64 rows (bounded partial traffic)
  const int64_t rows = std::max(h->NR, (int64_t)h->piece);
  h->chunk_rows = (int)std::max<int64_t>(64, round_up((rows + 47) / 48, 64));
  h->nb = (int)((rows + h->chunk_rows - 1) / h->chunk_rows);
  h->part = dalloc<double>((size_t)h->nb * (M + 1) * KK);
  h->red = dalloc<double>((size_t)(M + 1) * KK + 8);
  h->counters = dalloc<unsigned>((size_t)M + 8);
  // one-GPU fast k-wide chain (tensor-core G / S, k2f_fused_t, k2b_v4)
  h->fast = !h->grid() && k1_tc_k(K);
  const bool grid_fast = h->grid() && (K == 16 || K == 32);
  if (grid_fast) h->W32 = dalloc<float>((size_t)M * 2 * KK);
  if (dense_gram_tc(h)) {
    // tensor-core G / S_t over the reduced P (sp_gram_tc): 512-row chunks so
    // the (m+1) x chunks items cover the GPU at cfg2-sized n
    h->gchunks = (int)std::max<int64_t>(1, std::min<int64_t>(64, (h->rows_valid + 511) / 512));
    h->gpart = dalloc<double>((size_t)(M + 1) * h->gchunks * KK);
    RK_CUDA(cudaFuncSetAttribute(sp_gram_tc_of(K), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)rk::sp::SpGramTc::smem));
  }
  if (h->sparse) {
    h->numer = dalloc<double>((size_t)h->NR * K);
    h->gchunks = (int)std::max<int64_t>(1, std::min<int64_t>(64, (h->rows_valid + 2047) / 2048));
    h->gpart = dalloc<double>((size_t)(M + 1) * h->gchunks * KK);
    if (K == 16) {
      h->wfrag = dalloc<float4>((size_t)M * 256);
      RK_CUDA(cudaFuncSetAttribute(rk::sp::sp_numer_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)rk::sp::SpNumTc::smem));
      RK_CUDA(cudaFuncSetAttribute(rk::sp::sp_gram<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)rk::sp::SpGramCfg<16>::smem));
      RK_CUDA(cudaFuncSetAttribute(rk::sp::sp_gram_tc_k<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)rk::sp::SpGramTc::smem));
      RK_CUDA(cudaFuncSetAttribute(rk::sp::sp_numer_apply<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)rk::sp::SpNumCfg<16>::smem));
    } else {
      RK_CUDA(cudaFuncSetAttribute(rk::sp::sp_gram<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)rk::sp::SpGramCfg<32>::smem));
      RK_CUDA(cudaFuncSetAttribute(rk::sp::sp_numer_apply<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)rk::sp::SpNumCfg<32>::smem));
    }
    const size_t wsm = (size_t)M * 2 * KK * sizeof(float);
    // grid blocks keep the fused z-only CSC numerator (all W_t staged at once)
    RK_REQUIRE(!h->grid() || wsm <= 200 * 1024, RK_ERR_DATA,
               "sparse grid engine: m*k_pad^2 too large for the staged cores");
    if (h->grid()) {
      if (K == 16)
        RK_CUDA(cudaFuncSetAttribute(rk::sp::sp_csc_numer<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
      else
        RK_CUDA(cudaFuncSetAttribute(rk::sp::sp_csc_numer<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
    }
  }
  if (h->fast) {
    h->W32 = dalloc<float>((size_t)M * 2 * KK);
    std::vector<int> first(M), count(M, 1);
    for (int64_t t = 0; t < M; ++t) first[t] = (int)t;
    h->d_simt_first = dalloc<int>(M);
    h->d_simt_count = dalloc<int>(M);
    RK_CUDA(cudaMemcpy(h->d_simt_first, first.data(), sizeof(int) * M, cudaMemcpyHostToDevice));
    RK_CUDA(cudaMemcpy(h->d_simt_count, count.data(), sizeof(int) * M, cudaMemcpyHostToDevice));
  }
  if (!k2f_smem(K)) h->gscratch = dalloc<double>((size_t)M * 6 * KK);
  h->P = dalloc<float>((size_t)M * h->NR * K);
  h->Q = dalloc<float>((size_t)M * h->NC * K);
  h->nr = h->num_sms * 2;
  h->rpart = dalloc<double>(h->nr);
  h->regS = dalloc<double>(M * KK);
  h->regG = dalloc<double>(KK);
  h->regT = dalloc<double>(M * KK);
  h->regRn = dalloc<double>(M * KK);
  // engine
  int eng = h->requested_engine;
  if (h->sparse) eng = RK_ENGINE_SIMT;  // gather-bound CSR/CSC kernels (no GEMM reshaping)
  if (eng == RK_ENGINE_AUTO) eng = k1_tc_k(K) ? RK_ENGINE_TC : RK_ENGINE_SIMT;
  RK_REQUIRE(!(eng == RK_ENGINE_TC && !k1_tc_k(K)), RK_ERR_DATA,
             "tcgen05 engine needs k_pad in {16, 32, 48, 64}");
  h->engine = eng;
  if (eng == RK_ENGINE_TC) plan_tc(h);
  const size_t simt_smem = (size_t)(64 * 33 + 64 * K) * sizeof(float);
  RK_CUDA(cudaFuncSetAttribute(rk::k1_simt_p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)simt_smem));
  RK_CUDA(cudaFuncSetAttribute(rk::k1_simt_q, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)simt_smem));
  const size_t k5s = (size_t)(2 * 64 * (K + 1) + (K <= 128 ? K * K : 0)) * sizeof(float);
  RK_CUDA(cudaFuncSetAttribute(rk::k5_residual, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k5s));
  if (k2f_smem(K))
    RK_CUDA(cudaFuncSetAttribute(rk::k2f_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k2f_smem(K)));
  if (rk::k2b_fused_smem(K, (int)M) <= 200 * 1024)
    RK_CUDA(cudaFuncSetAttribute(rk::k2b_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)rk::k2b_fused_smem(K, (int)M)));
  RK_CUDA(cudaFuncSetAttribute(rk::k2a_gs, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * K * 8));
  if (K == 16 || K == 32) {
    if (K == 16) {
      RK_CUDA(cudaFuncSetAttribute(rk::k2a_v4<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      RK_CUDA(cudaFuncSetAttribute(rk::k2a_v4<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)rk::k2a_v4_smem(16)));
    } else {
      RK_CUDA(cudaFuncSetAttribute(rk::k2a_v4<32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      RK_CUDA(cudaFuncSetAttribute(rk::k2a_v4<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)rk::k2a_v4_smem(32)));
    }
    const int rbu = 2 * (256 / K);
    const int tgu = rk::k2b_u4_tg(K, (int)M);
    const int smu = tgu * (K * K + rbu * K) * (int)sizeof(float);
    if (K == 16)
      RK_CUDA(cudaFuncSetAttribute(rk::k2b_u4<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smu));
    else
      RK_CUDA(cudaFuncSetAttribute(rk::k2b_u4<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smu));
  }
  if (h->fast)
    RK_CUDA(cudaFuncSetAttribute(k2b_v4_of(K, rk::k2b_v4_rpt(K, h->NR)), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)rk::k2b_v4_smem(K, h->NR)));
  if (K == 48 || K == 64)
    RK_CUDA(cudaFuncSetAttribute(K == 48 ? rk::k2f_fused_t<48> : rk::k2f_fused_t<64>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k2f_smem(K)));
  const size_t k2bs = (size_t)(K <= 128 ? K * (K + 1) : 0) * 8 + 2 * (256 / K) * K * 4;
  RK_CUDA(cudaFuncSetAttribute(rk::k2b_update_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k2bs));
  const size_t k2ps = (size_t)K * (K + 1) * 8 + (256 / K) * K * 4;
  RK_CUDA(cudaFuncSetAttribute(rk::k2b_partial, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k2ps));
}

// ------------------------------- peer-memory grid exchange ------------------

void peer_teardown(rk_handle* h) {
  for (void* p : h->peer_open)
    if (p) cudaIpcCloseMemHandle(p);
  h->peer_open.clear();
  if (h->arena) cudaFree(h->arena);
  h->arena = nullptr;
  dfree(h->pep);
  h->pep = nullptr;
  h->peer = false;
}

// Collective over the world communicator (every rank calls it at the same
// point: the first rk_run after grid init / a rank change). Maps every rank's
// arena through CUDA IPC; any rank failing (no P2P path, RK_PEER=0) makes all
// ranks keep the NCCL schedule.
void ensure_peer(rk_handle* h) {
  if (!h->grid() || !(h->K == 16 || (h->K == 32 && !h->sparse)) || !h->W32) return;
  const int p = h->pr * h->pc;
  const int64_t key[4] = {h->K, h->m, h->piece, p};
  if (h->peer_tried && std::equal(key, key + 4, h->peer_key)) return;
  drop_graphs(h);
  peer_teardown(h);
  h->peer_tried = true;
  std::copy(key, key + 4, h->peer_key);
  // RK_PEER=0: NCCL, RK_PEER=1: peer memory, unset: peer memory while an A
  // piece is <= 16 MB. Larger pieces (the sparse cfg4 grid: 67 MB) move faster
  // through NCCL's copy protocols than through SM stores (measured 209 vs
  // 199 it/s on 1x2, profiles/r01s3_peer_sp1_*).
  static const int mode = [] {
    const char* e = std::getenv("RK_PEER");
    return e ? std::atoi(e) : -1;
  }();
  const int K = h->K;
  const int64_t b = h->piece;
  const bool disabled = mode == 0 || (mode < 0 && b * K * 8 > (16ll << 20));
  const int L = (int)((h->m + 1) * K * K + 1);
  auto al = [](int64_t v) { return round_up(v, 256); };
  rk::peer::Args& a = h->pargs;
  a = rk::peer::Args{};
  a.p = p;
  a.pr = h->pr;
  a.pc = h->pc;
  a.rank = h->rank;
  a.gi = h->gi;
  a.gj = h->gj;
  a.K = K;
  a.L = L;
  a.b = b;
  a.off_red = (long long)rk::peer::kFlagBytes;
  a.off_rxI = a.off_red + al((int64_t)2 * p * L * 8);
  a.off_rxJ = a.off_rxI + al((int64_t)2 * h->pc * b * K * 8);
  a.off_rxAr = a.off_rxJ + al((int64_t)2 * h->pr * b * K * 8);
  a.off_rxAc = a.off_rxAr + al((int64_t)2 * h->pc * b * K * 8);
  const size_t bytes = (size_t)(a.off_rxAc + al((int64_t)2 * h->pr * b * K * 8));
  int fail = (disabled || p > rk::peer::kMaxP) ? 1 : 0;
  cudaIpcMemHandle_t mine{};
  if (!fail && cudaMalloc(&h->arena, bytes) != cudaSuccess) {
    cudaGetLastError();
    h->arena = nullptr;
    fail = 1;
  }
  if (!fail && (cudaMemset(h->arena, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess ||
                cudaIpcGetMemHandle(&mine, h->arena) != cudaSuccess)) {
    cudaGetLastError();
    fail = 1;
  }
  // exchange the 64-byte handles over NCCL (stream-ordered, then read back)
  char* dh = dalloc<char>((size_t)p * sizeof(mine));
  int* dfail = dalloc<int>(1);
  std::vector<cudaIpcMemHandle_t> all(p);
  RK_CUDA(cudaMemcpy(dh + (size_t)h->rank * sizeof(mine), &mine, sizeof(mine), cudaMemcpyHostToDevice));
  RK_NCCL(ncclAllGather(dh + (size_t)h->rank * sizeof(mine), dh, sizeof(mine), ncclChar, h->world, h->stream));
  RK_CUDA(cudaStreamSynchronize(h->stream));
  RK_CUDA(cudaMemcpy(all.data(), dh, (size_t)p * sizeof(mine), cudaMemcpyDeviceToHost));
  h->peer_open.assign(p, nullptr);
  for (int r = 0; r < p && !fail; ++r) {
    if (r == h->rank) {
      a.base[r] = h->arena;
      continue;
    }
    void* ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, all[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      fail = 1;
      break;
    }
    h->peer_open[r] = ptr;
    a.base[r] = static_cast<char*>(ptr);
  }
  RK_CUDA(cudaMemcpy(dfail, &fail, sizeof(int), cudaMemcpyHostToDevice));
  RK_NCCL(ncclAllReduce(dfail, dfail, 1, ncclInt, ncclSum, h->world, h->stream));
  RK_CUDA(cudaStreamSynchronize(h->stream));
  int total = 0;
  RK_CUDA(cudaMemcpy(&total, dfail, sizeof(int), cudaMemcpyDeviceToHost));
  dfree(dh);
  dfree(dfail);
  if (total) {
    peer_teardown(h);
    return;
  }
  // k2b_u4's 48 KB staging + the ticket word exceed the default dynamic limit
  RK_CUDA(cudaFuncSetAttribute(rk::peer::k2b_u4_peer<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
  RK_CUDA(cudaFuncSetAttribute(rk::peer::k2b_u4_peer<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
  h->pep = dalloc<unsigned>(8);
  a.ep = h->pep;
  a.ctl = h->ctl;
  h->peer = true;
}

// Programmatic dependent launch (the kernel starts with rk::pdl_entry):
// the next kernel's launch overlaps this one's tail (graph edges become
// programmatic). Off unless RK_PDL=1: measured +0.25 % on cfg2 / +0.4 % on
// cfg3 and -5 % on the launch-bound cfg1 (profiles/r01s3_pdl_ab.txt).
bool pdl_on() {
  static const bool on = [] {
    const char* e = std::getenv("RK_PDL");
    return e && std::atoi(e) == 1;
  }();
  return on;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  RK_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// Launch as a cooperative grid: every CTA co-resident. K1 with strip groups
// needs it -- group members wait for each other's P tiles, which is only safe
// when all of them run at once, also next to another engine's kernels on the
// same GPU (a grid of one CTA per SM always fits an otherwise idle GPU).
template <typename... KArgs, typename... Args>
void launch_coop(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                 Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 2 : 1;
  RK_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// ------------------------------- launches ----------------------------------

void launch_k1(rk_handle* h, bool timed) {
  cudaStream_t s = h->stream;
  const int K = h->K, M = (int)h->m;
  if (timed) {
    size_t i = (size_t)h->k1_count * 2;
    if (h->ev_k1.size() < i + 2) {
      for (int q = 0; q < 2; ++q) {
        cudaEvent_t e;
        RK_CUDA(cudaEventCreate(&e));
        h->ev_k1.push_back(e);
      }
    }
    RK_CUDA(cudaEventRecord(h->ev_k1[i], s));
  }
  if (h->sparse) {
    const int grid = h->num_sms * 16;
    if (K == 16)
      rk::sp::sp_csr_pass<16><<<grid, 256, 0, s>>>(h->ctl, h->csr_ptr, h->csr_idx, h->csr_val, h->A32col,
                                                  h->P, (int)h->rows_valid, (int)h->NR, M, 1);
    else
      rk::sp::sp_csr_pass<32><<<grid, 256, 0, s>>>(h->ctl, h->csr_ptr, h->csr_idx, h->csr_val, h->A32col,
                                                  h->P, (int)h->rows_valid, (int)h->NR, M, 1);
    RK_CUDA(cudaGetLastError());
    if (timed) RK_CUDA(cudaEventRecord(h->ev_k1[(size_t)h->k1_count * 2 + 1], s));
    h->launches += 1;
  } else if (h->engine == RK_ENGINE_TC) {
    rk::tc::K1Args a;
    a.NR = (int)h->NR;
    a.NC = (int)h->NC;
    a.K = K;
    a.M = M;
    a.c = h->c;
    a.nstrips = h->nstrips;
    a.nrb = (int)(h->NR / 128);
    a.ncb = (int)(h->NC / 128);
    a.qrot = h->qrot;
    a.grp = h->k1_grp;
    a.sw = h->sw;
    a.Pscr = h->Pscr;
    a.pflag = h->pflag;
    a.Ppart = h->Ppart;
    a.Qpart = h->Qpart;
    a.cta_begin = h->d_cta_begin;
    a.cta_slot = h->d_cta_slot;
    a.ctl = h->ctl;
    a.skip_if_stopped = 1;
    if (h->k1_grp > 1)  // strip-group members wait for each other: co-resident grid
      launch_coop(k1_kernel_of(h), dim3(h->grid_tc), dim3(rk::tc::kThreads), h->smem_tc, s, h->maps[0],
                  h->maps[1], h->maps[2], h->maps[3], h->maps[4], h->maps[5], a);
    else
      launch_pdl(k1_kernel_of(h), dim3(h->grid_tc), dim3(rk::tc::kThreads), h->smem_tc, s, h->maps[0],
                 h->maps[1], h->maps[2], h->maps[3], h->maps[4], h->maps[5], a);
    RK_CUDA(cudaGetLastError());
    if (timed) RK_CUDA(cudaEventRecord(h->ev_k1[(size_t)h->k1_count * 2 + 1], s));
    h->launches += 1;
    {
      launch_pdl(rk::tc::k1_reduce, dim3(h->num_sms * 8), dim3(256), 0, s, (const Ctl*)h->ctl,
                 (const float*)h->Ppart, (const float*)h->Qpart, (const int*)h->d_slot_first,
                 (const int*)h->d_slot_count, h->P, h->Q, (int)h->NR, (int)h->NC, K, M, h->c, h->nstrips, 1,
                 h->sw, h->k1_grp);
      h->launches += 1;
    }
  } else {
    const size_t smem = (size_t)(64 * 33 + 64 * K) * sizeof(float);
    rk::k1_simt_p<<<dim3((unsigned)(h->NR / 32), M), rk::kThreads, smem, s>>>(
        h->ctl, h->Xh, h->Xl, h->A32col, h->P, (int)h->NR, (int)h->NC, K, 1);
    rk::k1_simt_q<<<dim3((unsigned)(h->NC / 32), M), rk::kThreads, smem, s>>>(
        h->ctl, h->Xh, h->Xl, h->A32row, h->Q, (int)h->NR, (int)h->NC, K, 1);
    RK_CUDA(cudaGetLastError());
    if (timed) RK_CUDA(cudaEventRecord(h->ev_k1[(size_t)h->k1_count * 2 + 1], s));
    h->launches += 2;
  }
  if (timed) h->k1_count += 1;
}

void launch_k5(rk_handle* h, int gate) {
  if (h->sparse) return;  // the sparse trace uses the Gram identity (no dense residual)
  const int K = h->K;
  const size_t smem = (size_t)(2 * 64 * (K + 1) + (K <= 128 ? K * K : 0)) * sizeof(float);
  launch_pdl(rk::k5_residual, dim3(h->nr), dim3(rk::kThreads), smem, h->stream, (const Ctl*)h->ctl,
             (const __nv_bfloat16*)h->Xh, (const __nv_bfloat16*)h->Xl, (const float*)h->A32row,
             (const float*)h->A32col, (const double*)h->R, (int)h->NR, (int)h->NC, K, (int)h->m,
             (int)h->rows_valid, (int)h->cols_valid, h->rpart, gate);
  RK_CUDA(cudaGetLastError());
  h->launches += 1;
}

// One GPU, tensor-core G / S (dense K in {16, 32}, sparse K = 16): k2f sums
// the chunk partials itself (one launch less per iteration); regress_r and
// the grid all-reduce need the reduced [G, S_t] in `red` first.
bool k2f_reduces(const rk_handle* h) { return !h->grid() && h->gpart && (h->K == 16 || !h->sparse); }

void launch_k2a(rk_handle* h, int skip, bool for_k2f = true) {
  const int K = h->K;
  if (h->sparse && (!h->grid() || K == 16)) {
    // G = A^T A, S_t = A^T P_t streamed from the stored P (sparse.cuh sp_gram);
    // on a grid G runs over the rank's own piece of A, S_t over its row set
    const int grid = h->num_sms * 2;
    const float* aown = h->grid() ? h->A32row + (size_t)h->gj * h->piece * K : nullptr;
    const int nown = h->grid() ? (int)h->piece : 0;
    if (K == 16)
      rk::sp::sp_gram_tc_k<16><<<h->num_sms * rk::sp::SpGramTc::CPS, 256, rk::sp::SpGramTc::smem, h->stream>>>(
          h->ctl, h->A32row, h->P, (int)h->rows_valid, (int)h->NR, (int)h->m, h->gchunks, h->gpart, skip, aown,
          nown);
    else if (K == 16)
      rk::sp::sp_gram<16><<<grid, 256, rk::sp::SpGramCfg<16>::smem, h->stream>>>(
          h->ctl, h->A32row, h->P, (int)h->rows_valid, (int)h->NR, (int)h->m, h->gchunks, h->gpart, skip);
    else
      rk::sp::sp_gram<32><<<grid, 256, rk::sp::SpGramCfg<32>::smem, h->stream>>>(
          h->ctl, h->A32row, h->P, (int)h->rows_valid, (int)h->NR, (int)h->m, h->gchunks, h->gpart, skip);
    if (!(for_k2f && k2f_reduces(h) && K == 16)) {
      rk::sp::sp_gram_reduce<<<(unsigned)(h->m + 1), 256, 0, h->stream>>>(h->ctl, h->gpart, h->gchunks, K * K,
                                                                          h->red, skip);
      h->launches += 1;
    }
    RK_CUDA(cudaGetLastError());
    h->launches += 1;
    return;
  }
  if (dense_gram_tc(h) && h->gpart) {
    // on a grid G runs over the rank's own piece of A (as k2a_v4's aown), S_t over its row set
    const float* aown = h->grid() ? h->A32row + (size_t)h->gj * h->piece * K : nullptr;
    const int nown = h->grid() ? (int)h->piece : 0;
    sp_gram_tc_of(K)<<<h->num_sms * rk::sp::SpGramTc::CPS, 256, rk::sp::SpGramTc::smem, h->stream>>>(
        h->ctl, h->A32row, h->P, (int)h->rows_valid, (int)h->NR, (int)h->m, h->gchunks, h->gpart, skip, aown, nown);
    if (!(for_k2f && k2f_reduces(h))) {
      rk::sp::sp_gram_reduce<<<(unsigned)(h->m + 1), 256, 0, h->stream>>>(h->ctl, h->gpart, h->gchunks, K * K,
                                                                          h->red, skip);
      h->launches += 1;
    }
    RK_CUDA(cudaGetLastError());
    h->launches += 1;
    return;
  }
  if ((h->fast && K <= 32) || (h->grid() && (K == 16 || K == 32))) {
    const float* aown = h->grid() ? h->A32row + (size_t)h->gj * h->piece * K : h->A32row;
    const int nown = h->grid() ? (int)h->piece : (int)h->NR;
    // P/Q already reduced (k1_reduce / SIMT K1 / sparse CSR pass)
    const int ncta = 8;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ncta, (unsigned)(h->m + 1));
    cfg.blockDim = dim3(K == 16 ? 512 : 256);
    cfg.dynamicSmemBytes = rk::k2a_v4_smem(K);
    cfg.stream = h->stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ncta;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_on() ? 2 : 1;
    if (K == 16)
      RK_CUDA(cudaLaunchKernelEx(&cfg, rk::k2a_v4<16>, (const Ctl*)h->ctl, (const float*)h->A32row, aown, nown,
                                 (const float*)h->P, (int)h->NR, (int)h->m, h->red, skip));
    else
      RK_CUDA(cudaLaunchKernelEx(&cfg, rk::k2a_v4<32>, (const Ctl*)h->ctl, (const float*)h->A32row, aown, nown,
                                 (const float*)h->P, (int)h->NR, (int)h->m, h->red, skip));
    h->launches += 1;
    return;
  }
  const double* Aown = h->grid() ? h->Arow + (size_t)h->gj * h->piece * K : h->Arow;
  const int Nown = h->grid() ? (int)h->piece : (int)h->NR;
  rk::k2a_gs<<<dim3(h->nb, (unsigned)(h->m + 1)), rk::kThreads, 2 * 64 * K * sizeof(double), h->stream>>>(
      h->ctl, Aown, Nown, h->Arow, h->P, (int)h->NR, K, (int)h->m, h->chunk_rows, h->part, h->red,
      h->counters, skip);
  RK_CUDA(cudaGetLastError());
  h->launches += 1;
}

// On a grid: append the direct-residual scalar to the reduced [G, S_t] and
// all-reduce over the world communicator (the only fp64 all-reduce of the
// iteration; it returns identical bytes on every rank, so R stays replicated).
void grid_allreduce_parts(rk_handle* h, bool with_resid) {
  const int K = h->K;
  const int len = (int)((h->m + 1) * K * K);
  if (h->peer) {
    rk::peer::peer_allreduce<<<h->pr * h->pc, 512, 0, h->stream>>>(h->pargs, h->red, len, h->rpart,
                                                                     with_resid ? h->nr : 0);
    RK_CUDA(cudaGetLastError());
    h->launches += 1;
    return;
  }
  rk::sum_scalars<<<1, 256, 0, h->stream>>>(h->rpart, with_resid ? h->nr : 0, h->red + len);
  if (!h->skip_comm)
    RK_NCCL(ncclAllReduce(h->red, h->red, (size_t)len + 1, ncclDouble, ncclSum, h->world, h->stream));
  h->launches += 1;
}

// K2f + trace/commit; mode: 0 iteration, 1 tail, 2 update_r, 3 update_a
void launch_k2f(rk_handle* h, int mode) {
  const int K = h->K;
  const int len = (int)((h->m + 1) * K * K);
  const double* rres = h->grid() ? h->red + len : h->rpart;
  const int nres = h->grid() ? 1 : h->nr;
  // after a launch_k2a(for_k2f) on a one-GPU tensor-core G / S path the
  // chunk partials are still unreduced: k2f sums them
  const double* gpart = k2f_reduces(h) ? h->gpart : nullptr;
  if (!h->gscratch && k1_tc_k(K)) {
    auto kern = K == 16 ? rk::k2f_fused_t<16>
                : K == 32 ? rk::k2f_fused_t<32>
                : K == 48 ? rk::k2f_fused_t<48>
                          : rk::k2f_fused_t<64>;
    launch_pdl(kern, dim3((unsigned)h->m), dim3(rk::kThreads), k2f_smem(K), h->stream, h->ctl, h->red, h->R,
               h->Rnext, h->Mt, h->Mm, h->tt, rres, nres, h->trace_dev, (int)h->m, h->eps, mode,
               h->counters + h->m + 1, h->W32, gpart, h->gchunks);
  } else {
    launch_pdl(rk::k2f_fused, dim3((unsigned)h->m), dim3(rk::kThreads), k2f_smem(K), h->stream, h->ctl, h->red,
               h->R, h->Rnext, h->Mt, h->Mm, h->tt, rres, nres, h->trace_dev, K, (int)h->m, h->eps, mode,
               h->gscratch, h->counters + h->m + 1, h->W32, gpart, h->gchunks);
  }
  RK_CUDA(cudaGetLastError());
  h->launches += 1;
}

void launch_emit(rk_handle* h) {
  const int K = h->K;
  // the sparse engine reads only the fp32 copies (no tensor-core planes)
  rk::emit_operands<<<h->num_sms * 2, 256, 0, h->stream>>>(h->Arow, (int)h->NR, K, h->A32row,
                                                           h->sparse ? nullptr : h->ATh_row,
                                                           h->sparse ? nullptr : h->ATl_row);
  if (h->grid())
    rk::emit_operands<<<h->num_sms * 2, 256, 0, h->stream>>>(h->Acol, (int)h->NC, K, h->A32col,
                                                             h->sparse ? nullptr : h->ATh_col,
                                                             h->sparse ? nullptr : h->ATl_col);
  RK_CUDA(cudaGetLastError());
  h->launches += h->grid() ? 2 : 1;
}

// Grid: gather the owned pieces into the row / col operand sets.
void grid_allgather_a(rk_handle* h) {
  const size_t cnt = (size_t)h->piece * h->K;
  if (h->skip_comm) return;
  RK_NCCL(ncclGroupStart());
  RK_NCCL(ncclAllGather(h->Arow + (size_t)h->gj * cnt, h->Arow, cnt, ncclDouble, h->rowc, h->stream));
  RK_NCCL(ncclAllGather(h->Arow + (size_t)h->gj * cnt, h->Acol, cnt, ncclDouble, h->colc, h->stream));
  RK_NCCL(ncclGroupEnd());
}

void phase_mark(rk_handle* h, bool timed, int idx);

void launch_k2b(rk_handle* h) {
  const int K = h->K;
  const double eps_m = h->eps * (double)h->m;
  if (h->sparse && !h->grid()) {
    // Q_t = X_t^T A from the CSC arrays (same gather kernel as the CSR pass),
    // then the fused numerator + A update over the stored P and Q
    const int grid = h->num_sms * 16;
    const unsigned nb = (unsigned)h->num_sms * 2;  // persistent: two CTAs per SM
    if (K == 16) {
      rk::sp::sp_csr_pass<16><<<grid, 256, 0, h->stream>>>(h->ctl, h->csc_ptr, h->csc_idx, h->csc_val, h->A32row,
                                                          h->Q, (int)h->cols_valid, (int)h->NC, (int)h->m, 1);
      rk::sp::sp_wfrag<<<(unsigned)h->m, 256, 0, h->stream>>>(h->ctl, h->W32, h->wfrag, (int)h->m);
      rk::sp::sp_numer_tc<<<(unsigned)h->num_sms * 2, 256, rk::sp::SpNumTc::smem, h->stream>>>(
          h->ctl, h->Arow, h->A32row, h->P, h->Q, (int)h->NR, (int)h->NC, h->wfrag, h->Mm, (int)h->n,
          (int)h->m, eps_m);
      h->launches += 1;
    } else {
      rk::sp::sp_csr_pass<32><<<grid, 256, 0, h->stream>>>(h->ctl, h->csc_ptr, h->csc_idx, h->csc_val, h->A32row,
                                                          h->Q, (int)h->cols_valid, (int)h->NC, (int)h->m, 1);
      rk::sp::sp_numer_apply<32><<<nb, 256, rk::sp::SpNumCfg<32>::smem, h->stream>>>(
          h->ctl, h->Arow, h->A32row, h->P, h->Q, (int)h->NR, (int)h->NC, h->W32, h->Mm, (int)h->n, (int)h->m,
          eps_m);
    }
    RK_CUDA(cudaGetLastError());
    h->launches += 2;
    return;
  }
  if (h->fast) {
    const int rb = rk::k2b_v4_rb(K, h->NR);
    const unsigned blocks = (unsigned)((h->NR + rb - 1) / rb);
    launch_pdl(k2b_v4_of(K, rk::k2b_v4_rpt(K, h->NR)), dim3(blocks), dim3(rk::k2b_v4_threads(K)),
               rk::k2b_v4_smem(K, h->NR), h->stream, h->ctl, h->Arow, h->A32row, h->ATh_row, h->ATl_row,
               (const float*)h->P, (const float*)h->Q, (const float*)h->W32, (const double*)h->Mm, (int)h->NR,
               (int)h->m, 0, eps_m);
    RK_CUDA(cudaGetLastError());
    h->launches += 1;
    return;
  }
  if (!h->grid()) {
    const int rpb = 256 / K;
    if (rk::k2b_fused_smem(K, (int)h->m) <= 200 * 1024) {
      const int rows_fused = rk::k2b_fused_rows(K);
      rk::k2b_fused<<<(unsigned)((h->NR + rows_fused - 1) / rows_fused), rk::kThreads,
                      rk::k2b_fused_smem(K, (int)h->m), h->stream>>>(
          h->ctl, h->Arow, h->A32row, h->ATh_row, h->ATl_row, h->P, h->Q, h->R, h->Mm, (int)h->NR, K,
          (int)h->m, eps_m);
      RK_CUDA(cudaGetLastError());
      h->launches += 1;
      return;
    }
    const size_t smem = (size_t)(K <= 128 ? K * (K + 1) : 0) * 8 + 2 * rpb * K * 4;
    rk::k2b_update_a<<<(unsigned)((h->NR + rpb - 1) / rpb), rk::kThreads, smem, h->stream>>>(
        h->ctl, h->Arow, h->A32row, h->ATh_row, h->ATl_row, h->P, h->Q, h->R, h->Mm, (int)h->NR, K,
        (int)h->m, eps_m, 0);
    RK_CUDA(cudaGetLastError());
    h->launches += 1;
    return;
  }
  const int rpb = 256 / K;
  if (h->sparse && K == 16) {
    // Q_t = X_t^T A[I] from the block's CSC (gather kernel), then the row and
    // column numerator partials U_I = sum_t P_t R_t^T, U_J = sum_t Q_t R_t on
    // tensor cores (sp_numer_tc single-operand mode)
    rk::sp::sp_wfrag<<<(unsigned)h->m, 256, 0, h->stream>>>(h->ctl, h->W32, h->wfrag, (int)h->m);
    rk::sp::sp_csr_pass<16><<<h->num_sms * 16, 256, 0, h->stream>>>(h->ctl, h->csc_ptr, h->csc_idx, h->csc_val,
                                                                    h->A32row, h->Q, (int)h->cols_valid,
                                                                    (int)h->NC, (int)h->m, 1);
    rk::sp::sp_numer_tc<<<(unsigned)h->num_sms * 2, 256, rk::sp::SpNumTc::smem, h->stream>>>(
        h->ctl, h->Arow, h->A32row, h->P, nullptr, (int)h->NR, 0, h->wfrag, h->Mm, (int)h->rows_valid,
        (int)h->m, eps_m, 0, h->UI);
    rk::sp::sp_numer_tc<<<(unsigned)h->num_sms * 2, 256, rk::sp::SpNumTc::smem, h->stream>>>(
        h->ctl, h->Arow, h->A32row, h->Q, nullptr, (int)h->NC, 0, h->wfrag, h->Mm, (int)h->cols_valid,
        (int)h->m, eps_m, 1, h->UJ);
    h->launches += 3;
    if (h->peer) {
      // numerator rows -> owners' slots, owner update, pieces -> peers (peer.cuh)
      rk::peer::push_u_peer<<<h->num_sms * 4, 256, 0, h->stream>>>(h->ctl, h->UI, h->UJ, h->pargs);
      phase_mark(h, h->profile, 5);
      rk::peer::apply_peer<<<(unsigned)((h->piece + rpb - 1) / rpb), rk::kThreads, 0, h->stream>>>(
          h->ctl, h->Arow + (size_t)h->gj * h->piece * K, h->Mm, K, eps_m, h->pargs);
      rk::peer::emit_peer<<<h->num_sms * 2, rk::kThreads, 0, h->stream>>>(
          h->pargs, h->Arow, (int)h->NR, h->A32row, nullptr, nullptr, h->Acol, (int)h->NC, h->A32col, nullptr,
          nullptr);
      RK_CUDA(cudaGetLastError());
      h->launches += 3;
      return;
    }
  } else if (h->sparse) {
    // U_I = sum_t P_t R_t^T over the row set (dense P); U_J = sum_t z_t R_t with
    // z_t = X_t^T A_row streamed from the block's CSC (no P part: P_t lives on
    // the row set)
    const int rb = 2 * (256 / K);
    const int tg = rk::k2b_u4_tg(K, (int)h->m);
    const size_t smem = (size_t)tg * (K * K + rb * K) * sizeof(float);
    const size_t wsm = (size_t)h->m * 2 * K * K * sizeof(float);
    const int grid = h->num_sms * 4;
    if (K == 16) {
      rk::k2b_u4<16><<<(unsigned)((h->NR + rb - 1) / rb), 256, smem, h->stream>>>(h->ctl, h->P, h->W32, 0, (int)h->NR, (int)h->m, tg, h->UI);
      rk::sp::sp_csc_numer<16><<<grid, 512, wsm, h->stream>>>(h->ctl, h->csc_ptr, h->csc_idx, h->csc_val, h->A32row,
                                                              nullptr, h->W32, h->UJ, (int)h->cols_valid, (int)h->NC, (int)h->m);
    } else {
      rk::k2b_u4<32><<<(unsigned)((h->NR + rb - 1) / rb), 256, smem, h->stream>>>(h->ctl, h->P, h->W32, 0, (int)h->NR, (int)h->m, tg, h->UI);
      rk::sp::sp_csc_numer<32><<<grid, 512, wsm, h->stream>>>(h->ctl, h->csc_ptr, h->csc_idx, h->csc_val, h->A32row,
                                                              nullptr, h->W32, h->UJ, (int)h->cols_valid, (int)h->NC, (int)h->m);
    }
  } else if (h->W32 && h->peer) {
    // numerator rows straight into the owners' slots, owner update, pieces
    // straight into the peers' operand sets (peer.cuh): no NCCL calls
    const int rb = 2 * (256 / K);
    const int tg = rk::k2b_u4_tg(K, (int)h->m);
    const size_t smem = (size_t)tg * (K * K + rb * K) * sizeof(float);
    const dim3 gu((unsigned)((std::max(h->NR, h->NC) + rb - 1) / rb), 2);
    if (K == 16)
      rk::peer::k2b_u4_peer<16><<<gu, 256, smem, h->stream>>>(h->ctl, h->P, h->Q, h->W32, (int)h->NR,
                                                                (int)h->NC, (int)h->m, tg, h->pargs);
    else
      rk::peer::k2b_u4_peer<32><<<gu, 256, smem, h->stream>>>(h->ctl, h->P, h->Q, h->W32, (int)h->NR,
                                                                (int)h->NC, (int)h->m, tg, h->pargs);
    RK_CUDA(cudaGetLastError());
    phase_mark(h, h->profile, 5);
    rk::peer::apply_peer<<<(unsigned)((h->piece + rpb - 1) / rpb), rk::kThreads, 0, h->stream>>>(
        h->ctl, h->Arow + (size_t)h->gj * h->piece * K, h->Mm, K, eps_m, h->pargs);
    rk::peer::emit_peer<<<h->num_sms * 2, rk::kThreads, 0, h->stream>>>(
        h->pargs, h->Arow, (int)h->NR, h->A32row, h->ATh_row, h->ATl_row, h->Acol, (int)h->NC, h->A32col,
        h->ATh_col, h->ATl_col);
    RK_CUDA(cudaGetLastError());
    h->launches += 3;
    return;
  } else if (h->W32) {
    const int rb = 2 * (256 / K);
    const int tg = rk::k2b_u4_tg(K, (int)h->m);
    const size_t smem = (size_t)tg * (K * K + rb * K) * sizeof(float);
    if (K == 16) {
      rk::k2b_u4<16><<<(unsigned)((h->NR + rb - 1) / rb), 256, smem, h->stream>>>(h->ctl, h->P, h->W32, 0, (int)h->NR, (int)h->m, tg, h->UI);
      rk::k2b_u4<16><<<(unsigned)((h->NC + rb - 1) / rb), 256, smem, h->stream>>>(h->ctl, h->Q, h->W32, 1, (int)h->NC, (int)h->m, tg, h->UJ);
    } else {
      rk::k2b_u4<32><<<(unsigned)((h->NR + rb - 1) / rb), 256, smem, h->stream>>>(h->ctl, h->P, h->W32, 0, (int)h->NR, (int)h->m, tg, h->UI);
      rk::k2b_u4<32><<<(unsigned)((h->NC + rb - 1) / rb), 256, smem, h->stream>>>(h->ctl, h->Q, h->W32, 1, (int)h->NC, (int)h->m, tg, h->UJ);
    }
  } else {
    const size_t smem = (size_t)K * (K + 1) * 8 + rpb * K * 4;
    rk::k2b_partial<<<(unsigned)((h->NR + rpb - 1) / rpb), rk::kThreads, smem, h->stream>>>(
        h->ctl, h->P, h->R, (int)h->NR, K, (int)h->m, 1, h->UI);
    rk::k2b_partial<<<(unsigned)((h->NC + rpb - 1) / rpb), rk::kThreads, smem, h->stream>>>(
        h->ctl, h->Q, h->R, (int)h->NC, K, (int)h->m, 0, h->UJ);
  }
  RK_CUDA(cudaGetLastError());
  const size_t cnt = (size_t)h->piece * K;
  // reduce-scatter in place: the own piece's sum lands at its slot; the row
  // and col collectives are independent -> one NCCL group
  if (!h->skip_comm) {
  RK_NCCL(ncclGroupStart());
  RK_NCCL(ncclReduceScatter(h->UI, h->UI + (size_t)h->gj * cnt, cnt, ncclDouble, ncclSum, h->rowc,
                            h->stream));
  RK_NCCL(ncclReduceScatter(h->UJ, h->UJ + (size_t)h->gi * cnt, cnt, ncclDouble, ncclSum, h->colc,
                            h->stream));
  RK_NCCL(ncclGroupEnd());
  }
  phase_mark(h, h->profile, 5);
  rk::k2b_apply_own<<<(unsigned)((h->piece + rpb - 1) / rpb), rk::kThreads, 0, h->stream>>>(
      h->ctl, h->Arow + (size_t)h->gj * cnt, h->UI + (size_t)h->gj * cnt, h->UJ + (size_t)h->gi * cnt,
      h->Mm, (int)h->piece, K, eps_m);
  RK_CUDA(cudaGetLastError());
  grid_allgather_a(h);
  launch_emit(h);
  h->launches += 3;
}

void phase_mark(rk_handle* h, bool timed, int idx) {
  if (!timed) return;
  const size_t i = (size_t)h->ph_iters * (rk_handle::kPhases + 1) + idx;
  while (h->ev_ph.size() <= i) {
    cudaEvent_t e;
    RK_CUDA(cudaEventCreate(&e));
    h->ev_ph.push_back(e);
  }
  RK_CUDA(cudaEventRecord(h->ev_ph[i], h->stream));
}

// NVTX ranges with the reference's phase names (grid.py:97-111 counted_mm
// phases, perf.py:32-33) around the host enqueue of each phase; emitted only
// in profile mode (per-phase events, no graph replay), so a timeline tool
// shows matrix_mul / gram_mul / row_reduce ... next to the kernels.
struct NvtxPhase {
  bool on;
  NvtxPhase(bool enable, const char* name) : on(enable) {
    if (on) nvtxRangePushA(name);
  }
  ~NvtxPhase() {
    if (on) nvtxRangePop();
  }
};

// phases: 0 K1(+reduce) | 1 K5+K2a | 2 grid all-reduce | 3 K2f | 4 K2b/numerator (+RS) | 5 A update/gather
void enqueue_iteration(rk_handle* h, bool timed, bool with_k5) {
  phase_mark(h, timed, 0);
  {
    NvtxPhase r(timed, h->sparse ? "matrix_mul_sparse" : "matrix_mul");
    launch_k1(h, timed);
  }
  phase_mark(h, timed, 1);
  {
    NvtxPhase r(timed, "gram_mul");
    if (with_k5) launch_k5(h, 1);
    launch_k2a(h, 1);
  }
  phase_mark(h, timed, 2);
  if (h->grid()) {
    NvtxPhase r(timed, "column_reduce");
    grid_allreduce_parts(h, true);
  }
  phase_mark(h, timed, 3);
  {
    NvtxPhase r(timed, "matrix_mul");
    launch_k2f(h, 0);
  }
  phase_mark(h, timed, 4);
  {
    NvtxPhase r(timed, h->grid() ? "row_reduce" : "matrix_mul");
    launch_k2b(h);
  }
  phase_mark(h, timed, 6);
  if (timed) h->ph_iters += 1;
}

void enqueue_tail(rk_handle* h) {
  rk::set_tail<<<1, 1, 0, h->stream>>>(h->ctl, 1);
  launch_k1(h, false);
  launch_k5(h, 1);
  launch_k2a(h, 1);
  if (h->grid()) grid_allreduce_parts(h, true);
  launch_k2f(h, 1);
}

void reset_ctl(rk_handle* h, int track, double tol, int max_iters) {
  Ctl c;
  std::memset(&c, 0, sizeof(c));
  c.track = track;
  c.tol = tol;
  c.eps = h->eps;
  c.norm2 = h->norm2;
  c.norm2_dev = h->norm2_dev;
  c.direct_thresh = h->sparse ? -1.0 : 0.2;
  c.max_iters = max_iters;
  *h->ctl_host = c;
  RK_CUDA(cudaMemcpyAsync(h->ctl, h->ctl_host, sizeof(Ctl), cudaMemcpyHostToDevice, h->stream));
}

void read_ctl(rk_handle* h) {
  RK_CUDA(cudaMemcpyAsync(h->ctl_host, h->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream));
  RK_CUDA(cudaStreamSynchronize(h->stream));
}

void ensure_trace(rk_handle* h, int cap) {
  if (cap + 1 > h->trace_cap) {
    drop_graphs(h);  // the captured trace/commit nodes hold the old pointer
    dfree(h->trace_dev);
    h->trace_cap = cap + 1;
    h->trace_dev = dalloc<double>(h->trace_cap);
  }
}

void check_ready(rk_handle* h) {
  RK_REQUIRE(h != nullptr, RK_ERR_DATA, "null handle");
  RK_REQUIRE(h->have_x, RK_ERR_DATA, "no tensor uploaded");
  RK_CUDA(cudaSetDevice(h->dev));
}

void finish_upload_norm(rk_handle* h, bool exact_from_dev) {
  std::vector<double> p(h->nnp), p2(h->nnp);
  RK_CUDA(cudaStreamSynchronize(h->stream));
  RK_CUDA(cudaMemcpy(p.data(), h->npart, sizeof(double) * h->nnp, cudaMemcpyDeviceToHost));
  RK_CUDA(cudaMemcpy(p2.data(), h->npart2, sizeof(double) * h->nnp, cudaMemcpyDeviceToHost));
  double s = 0.0, s2 = 0.0;
  for (int i = 0; i < h->nnp; ++i) {
    s += p[i];
    s2 += p2[i];
  }
  h->norm2_dev = s;
  if (exact_from_dev) h->norm2 = s2;
  if (h->grid()) {
    double v[2] = {h->norm2_dev, exact_from_dev ? h->norm2 : 0.0};
    double* d = h->red;
    RK_CUDA(cudaMemcpy(d, v, sizeof(v), cudaMemcpyHostToDevice));
    RK_NCCL(ncclAllReduce(d, d, 2, ncclDouble, ncclSum, h->world, h->stream));
    RK_CUDA(cudaStreamSynchronize(h->stream));
    RK_CUDA(cudaMemcpy(v, d, sizeof(v), cudaMemcpyDeviceToHost));
    h->norm2_dev = v[0];
    if (exact_from_dev) h->norm2 = v[1];
  }
  h->norm2_dev0 = h->norm2_dev;
}

void set_block_dims(rk_handle* h, int64_t rows_valid, int64_t cols_valid, int64_t NR, int64_t NC) {
  h->rows_valid = rows_valid;
  h->cols_valid = cols_valid;
  h->NR = NR;
  h->NC = NC;
}

void alloc_tensor(rk_handle* h) {
  if (h->sparse) return;
  dfree(h->Xh);
  dfree(h->Xl);
  dfree(h->Xh0);
  dfree(h->Xl0);
  h->Xh0 = h->Xl0 = nullptr;
  const size_t count = (size_t)h->m * h->NR * h->NC;
  h->Xh = dalloc<__nv_bfloat16>(count);
  h->Xl = dalloc<__nv_bfloat16>(count);
}

// A new tensor invalidates the unperturbed base copies rk_perturb keeps (they
// are re-taken from the new tensor at the next rk_perturb).
void drop_base_copies(rk_handle* h) {
  dfree(h->Xh0);
  dfree(h->Xl0);
  dfree(h->csr_val0);
  dfree(h->csc_val0);
  h->Xh0 = h->Xl0 = nullptr;
  h->csr_val0 = h->csc_val0 = nullptr;
}

// memcpy on up to 16 host threads (a pageable caller buffer -> pinned stage:
// one thread moves ~5-10 GB/s, the H2D copy behind it ~50 GB/s)
void parallel_memcpy(void* dst, const void* src, size_t bytes) {
  const size_t min_part = 4ull << 20;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t parts = std::min<size_t>(std::min<size_t>(hw, 16), std::max<size_t>(1, bytes / min_part));
  if (parts <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t per = (bytes + parts - 1) / parts;
  std::vector<std::thread> th;
  for (size_t i = 1; i < parts; ++i) {
    const size_t o = i * per;
    if (o >= bytes) break;
    th.emplace_back([=] {
      std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, std::min(per, bytes - o));
    });
  }
  std::memcpy(dst, src, std::min(per, bytes));
  for (auto& t : th) t.join();
}

template <typename T>
void upload_rows(rk_handle* h, const T* x, int64_t rows, int64_t cols) {
  // chunks of host rows through a pinned staging ring when the host buffer is
  // pageable; straight async copies when it is already pinned. The copies run
  // on their own stream, the split kernels on the handle's: the split of
  // chunk i overlaps the copy of chunk i + 1 (a copy-bound upload), ordered
  // by events per staging slot, without host waits for a pinned source.
  cudaPointerAttributes attr;
  bool pinned = cudaPointerGetAttributes(&attr, x) == cudaSuccess &&
                (attr.type == cudaMemoryTypeHost);
  cudaGetLastError();
  const size_t row_bytes = (size_t)cols * sizeof(T);
  const size_t chunk_bytes = 64ull << 20;
  const int64_t rows_per = std::max<int64_t>(1, (int64_t)(chunk_bytes / row_bytes));
  T* dstage[2] = {dalloc<T>((size_t)rows_per * cols), dalloc<T>((size_t)rows_per * cols)};
  T* hstage[2] = {nullptr, nullptr};
  if (!pinned)
    for (int i = 0; i < 2; ++i) RK_CUDA(cudaMallocHost(&hstage[i], (size_t)rows_per * row_bytes));
  cudaStream_t cs;
  RK_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaEvent_t copied[2], split[2];
  for (int i = 0; i < 2; ++i) {
    RK_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
    RK_CUDA(cudaEventCreateWithFlags(&split[i], cudaEventDisableTiming));
  }
  RK_CUDA(cudaEventRecord(split[0], h->stream));  // the upload starts after the handle's pending work
  RK_CUDA(cudaStreamWaitEvent(cs, split[0], 0));
  bool used[2] = {false, false};
  int slot = 0;
  for (int64_t t = 0; t < h->m; ++t) {
    for (int64_t r0 = 0; r0 < rows; r0 += rows_per) {
      const int64_t nrow = std::min(rows_per, rows - r0);
      const T* src = x + ((size_t)t * rows + r0) * cols;
      const T* from = src;
      if (!pinned) {
        if (used[slot]) RK_CUDA(cudaEventSynchronize(copied[slot]));  // host staging slot free
        parallel_memcpy(hstage[slot], src, (size_t)nrow * row_bytes);
        from = hstage[slot];
      }
      if (used[slot]) RK_CUDA(cudaStreamWaitEvent(cs, split[slot], 0));  // device staging slot free
      RK_CUDA(cudaMemcpyAsync(dstage[slot], from, (size_t)nrow * row_bytes, cudaMemcpyHostToDevice, cs));
      RK_CUDA(cudaEventRecord(copied[slot], cs));
      RK_CUDA(cudaStreamWaitEvent(h->stream, copied[slot], 0));
      rk::split_chunk<T><<<h->nnp, rk::kThreads, 0, h->stream>>>(
          dstage[slot], nrow, cols, h->Xh, h->Xl, h->NR, h->NC, (int)t, r0, h->npart, h->npart2);
      RK_CUDA(cudaGetLastError());
      RK_CUDA(cudaEventRecord(split[slot], h->stream));
      used[slot] = true;
      slot ^= 1;
    }
  }
  RK_CUDA(cudaStreamSynchronize(h->stream));
  RK_CUDA(cudaStreamSynchronize(cs));
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(copied[i]);
    cudaEventDestroy(split[i]);
    dfree(dstage[i]);
    if (hstage[i]) cudaFreeHost(hstage[i]);
  }
  cudaStreamDestroy(cs);
}

void regress_core(rk_handle* h, int max_iters, double tol, double eps, int* iters_done) {
  // S_t = A^T X_t A with the handle's A (one contraction pass), then sweeps.
  const int K = h->K;
  reset_ctl(h, 0, -1.0, 0);
  launch_k1(h, false);
  launch_k2a(h, 0, false);
  if (h->grid()) grid_allreduce_parts(h, false);
  rk::regress_loop<<<1, 1024, 0, h->stream>>>(h->red, 1, h->R, h->regS, h->regG, h->regT, h->regRn,
                                             K, (int)h->m, eps, max_iters, tol, h->d_iters);
  RK_CUDA(cudaGetLastError());
  RK_CUDA(cudaStreamSynchronize(h->stream));
  int it = 0;
  RK_CUDA(cudaMemcpy(&it, h->d_iters, sizeof(int), cudaMemcpyDeviceToHost));
  if (iters_done) *iters_done = it;
}

}  // namespace

namespace {
// Shared tail of the CSR uploads: build the CSC copy on the device. The
// block has `rows` CSR rows and `cols` columns per slice.
// bounds[t] = first stored entry of slice t, bounds[M] = nnz.
void build_csc(rk_handle* h, const std::vector<int64_t>& bounds) {
  const int64_t rows = h->rows_valid, cols = h->cols_valid, M = h->m;
  int64_t max_nnz = 0;
  for (int64_t t = 0; t < M; ++t)
    max_nnz = std::max(max_nnz, bounds[t + 1] - bounds[t]);
  uint64_t* keys = dalloc<uint64_t>((size_t)std::max<int64_t>(1, max_nnz));
  uint64_t* keys2 = dalloc<uint64_t>((size_t)std::max<int64_t>(1, max_nnz));
  int* counts = dalloc<int>((size_t)cols);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, h->csr_val, h->csc_val,
                                  (int)std::max<int64_t>(1, max_nnz), 0, 64, h->stream);
  void* tmp = dalloc<uint8_t>(tmp_bytes + 16);
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, scan_bytes, counts, h->csc_ptr, cub::Sum(), (int64_t)0, (int)cols,
                                 h->stream);
  void* scan_tmp = dalloc<uint8_t>(scan_bytes + 16);
  // the last offset of each slice comes from host memory that outlives the
  // asynchronous copies (filled before each copy is enqueued)
  std::vector<int64_t> ends((size_t)M);
  for (int64_t t = 0; t < M; ++t) {
    const int64_t base = bounds[t], cnt = bounds[t + 1] - base;
    RK_CUDA(cudaMemsetAsync(counts, 0, sizeof(int) * cols, h->stream));
    if (cnt > 0) {
      rk::sp::sp_make_keys<<<h->num_sms * 4, 256, 0, h->stream>>>(h->csr_ptr + t * (rows + 1), h->csr_idx,
                                                                   (int)rows, base, cnt, keys);
      const int bits = 32 + (int)std::ceil(std::log2((double)std::max<int64_t>(2, cols)));
      RK_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, h->csr_val + base,
                                              h->csc_val + base, (int)cnt, 0, std::min(64, bits),
                                              h->stream));
      rk::sp::sp_split_keys<<<h->num_sms * 4, 256, 0, h->stream>>>(keys2, cnt, h->csc_idx + base, counts);
    }
    RK_CUDA(cub::DeviceScan::ExclusiveScan(scan_tmp, scan_bytes, counts, h->csc_ptr + t * (cols + 1),
                                           cub::Sum(), (int64_t)base, (int)cols, h->stream));
    ends[t] = base + cnt;
    RK_CUDA(cudaMemcpyAsync(h->csc_ptr + t * (cols + 1) + cols, &ends[t], sizeof(int64_t),
                            cudaMemcpyHostToDevice, h->stream));
    RK_CUDA(cudaGetLastError());
  }
  RK_CUDA(cudaStreamSynchronize(h->stream));
  dfree(keys);
  dfree(keys2);
  dfree(counts);
  dfree(tmp);
  dfree(scan_tmp);
}

// ||X||^2 over all ranks (the trace denominator is global)
double global_sum(rk_handle* h, double v) {
  if (!h->grid()) return v;
  double* d = h->red;
  RK_CUDA(cudaMemcpy(d, &v, sizeof(double), cudaMemcpyHostToDevice));
  RK_NCCL(ncclAllReduce(d, d, 1, ncclDouble, ncclSum, h->world, h->stream));
  RK_CUDA(cudaStreamSynchronize(h->stream));
  RK_CUDA(cudaMemcpy(&v, d, sizeof(double), cudaMemcpyDeviceToHost));
  return v;
}
}  // namespace

// =============================== C ABI ======================================

namespace {
// Host -> device streaming through a pinned two-slot ring: pageable sources
// are copied into the pinned slot by several host threads while the other
// slot's DMA and post-processing kernel run (pinned sources are DMA'd
// directly). `post(dev_chunk, offset, bytes)` runs on the stream after each
// chunk has landed in `dev_dst + offset` (or in a device staging slot when
// dev_dst is null).
class Uploader {
 public:
  static constexpr size_t kChunk = 64ull << 20;
  explicit Uploader(rk_handle* h) : h_(h) {
    for (int i = 0; i < 2; ++i) {
      RK_CUDA(cudaMallocHost(&host_[i], kChunk));
      dev_[i] = dalloc<uint8_t>(kChunk);
      RK_CUDA(cudaEventCreateWithFlags(&done_[i], cudaEventDisableTiming));
    }
    const unsigned hw = std::thread::hardware_concurrency();
    threads_ = (int)std::max(1u, std::min(8u, hw ? hw : 1u));
  }
  ~Uploader() {
    cudaStreamSynchronize(h_->stream);
    for (int i = 0; i < 2; ++i) {
      cudaFreeHost(host_[i]);
      dfree(dev_[i]);
      cudaEventDestroy(done_[i]);
    }
  }
  double wait_ms = 0.0, memcpy_ms = 0.0;  // diagnostics
  template <typename Post>
  void copy(const void* src, size_t bytes, void* dev_dst, Post post) {
    cudaPointerAttributes attr;
    const bool pinned = cudaPointerGetAttributes(&attr, src) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();
    for (size_t off = 0; off < bytes; off += kChunk) {
      const size_t nb = std::min(kChunk, bytes - off);
      auto t0 = std::chrono::steady_clock::now();
      if (used_[slot_]) RK_CUDA(cudaEventSynchronize(done_[slot_]));
      auto t1 = std::chrono::steady_clock::now();
      const uint8_t* from = static_cast<const uint8_t*>(src) + off;
      if (!pinned) {
        par_memcpy(host_[slot_], from, nb);
        from = host_[slot_];
      }
      auto t2 = std::chrono::steady_clock::now();
      wait_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
      memcpy_ms += std::chrono::duration<double, std::milli>(t2 - t1).count();
      uint8_t* to = dev_dst ? static_cast<uint8_t*>(dev_dst) + off : dev_[slot_];
      RK_CUDA(cudaMemcpyAsync(to, from, nb, cudaMemcpyHostToDevice, h_->stream));
      post(to, off, nb);
      RK_CUDA(cudaGetLastError());
      RK_CUDA(cudaEventRecord(done_[slot_], h_->stream));
      used_[slot_] = true;
      slot_ ^= 1;
    }
  }

 private:
  void par_memcpy(void* dst, const void* src, size_t nb) {
    const size_t min_part = 4ull << 20;
    const int nt = (int)std::min<size_t>(threads_, std::max<size_t>(1, nb / min_part));
    if (nt <= 1) {
      std::memcpy(dst, src, nb);
      return;
    }
    std::vector<std::thread> th;
    const size_t part = (nb + nt - 1) / nt;
    for (int i = 0; i < nt; ++i) {
      const size_t o = (size_t)i * part;
      if (o >= nb) break;
      th.emplace_back([=] {
        std::memcpy(static_cast<uint8_t*>(dst) + o, static_cast<const uint8_t*>(src) + o, std::min(part, nb - o));
      });
    }
    for (auto& t : th) t.join();
  }
  rk_handle* h_;
  uint8_t* host_[2] = {nullptr, nullptr};
  uint8_t* dev_[2] = {nullptr, nullptr};
  cudaEvent_t done_[2];
  bool used_[2] = {false, false};
  int slot_ = 0;
  int threads_ = 1;
};

// Shared body of the CSR uploads: per-slice host arrays (local indptr,
// indices, values) -> device CSR with global offsets, validated and
// converted on the device, then the device-built CSC.
void upload_csr_slices(rk_handle* h, const int64_t* const* indptrs, const int32_t* const* indices,
                       const void* const* data, const int64_t* nnz_t, int32_t dtype) {
  static const bool timing = std::getenv("RK_UPLOAD_TIMING") != nullptr;  // diagnostics only
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t_start = now();
  auto ms_since = [&](std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double, std::milli>(now() - a).count();
  };
  const int64_t rows = h->rows_valid, cols = h->cols_valid, M = h->m;
  RK_REQUIRE(dtype == RK_F32 || dtype == RK_F64, RK_ERR_DATA, "unsupported dtype");
  std::vector<int64_t> bounds((size_t)M + 1, 0);
  int64_t nnz = 0;
  for (int64_t t = 0; t < M; ++t) {
    RK_REQUIRE(indptrs[t] != nullptr, RK_ERR_DATA, "null indptr");
    RK_REQUIRE(nnz_t[t] >= 0 && indptrs[t][0] == 0 && indptrs[t][rows] == nnz_t[t], RK_ERR_DATA,
               "inconsistent indptr");
    RK_REQUIRE(nnz_t[t] == 0 || (indices[t] && data[t]), RK_ERR_DATA, "null argument");
    nnz += nnz_t[t];
    bounds[(size_t)t + 1] = nnz;
  }
  void* old[] = {h->csr_ptr, h->csc_ptr, h->csr_idx, h->csc_idx, h->csr_val, h->csc_val, h->csr_val0,
                 h->csc_val0};
  for (void* p : old) dfree(p);
  h->csr_val0 = h->csc_val0 = nullptr;
  h->nnz = nnz;
  h->csr_ptr = dalloc<int64_t>((size_t)M * (rows + 1));
  h->csc_ptr = dalloc<int64_t>((size_t)M * (cols + 1));
  h->csr_idx = dalloc<int>((size_t)std::max<int64_t>(1, nnz));
  h->csc_idx = dalloc<int>((size_t)std::max<int64_t>(1, nnz));
  h->csr_val = dalloc<float>((size_t)std::max<int64_t>(1, nnz));
  h->csc_val = dalloc<float>((size_t)std::max<int64_t>(1, nnz));
  const size_t vsize = dtype == RK_F32 ? 4 : 8;
  const size_t nchunks = (size_t)(nnz * vsize / Uploader::kChunk) + (size_t)M + 2;
  const int pblocks = h->num_sms * 2;
  double* part = dalloc<double>(nchunks * pblocks);
  int* flag = dalloc<int>(1);
  RK_CUDA(cudaMemsetAsync(part, 0, sizeof(double) * nchunks * pblocks, h->stream));
  RK_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), h->stream));
  size_t chunk_id = 0;
  const double t_setup = ms_since(t_start);
  {
    Uploader up(h);
    int64_t base = 0;
    for (int64_t t = 0; t < M; ++t) {
      int64_t* dptr = h->csr_ptr + t * (rows + 1);
      up.copy(indptrs[t], sizeof(int64_t) * (rows + 1), nullptr, [&](void* d, size_t off, size_t nb) {
        rk::sp::sp_rebase_ptr<<<h->num_sms * 2, 256, 0, h->stream>>>(
            static_cast<const int64_t*>(d), (int64_t)(nb / 8), base, dptr + off / 8);
      });
      if (nnz_t[t] > 0) {
        up.copy(indices[t], sizeof(int32_t) * nnz_t[t], h->csr_idx + base, [&](void* d, size_t, size_t nb) {
          rk::sp::sp_check_idx<<<h->num_sms * 2, 256, 0, h->stream>>>(static_cast<const int*>(d),
                                                                      (int64_t)(nb / 4), (int)cols, flag);
        });
        float* vdst = h->csr_val + base;
        up.copy(data[t], vsize * nnz_t[t], dtype == RK_F32 ? (void*)vdst : nullptr,
                [&](void* d, size_t off, size_t nb) {
                  double* pp = part + (chunk_id++) * pblocks;
                  if (dtype == RK_F32)
                    rk::sp::sp_take_vals<float><<<pblocks, 256, 0, h->stream>>>(
                        static_cast<const float*>(d), (int64_t)(nb / 4), vdst + off / 4, pp, flag);
                  else
                    rk::sp::sp_take_vals<double><<<pblocks, 256, 0, h->stream>>>(
                        static_cast<const double*>(d), (int64_t)(nb / 8), vdst + off / 8, pp, flag);
                });
      }
      base += nnz_t[t];
    }
    if (timing)
      std::fprintf(stderr, "[rk]   ring: host memcpy %.1f ms, slot waits %.1f ms, setup %.1f ms\n", up.memcpy_ms,
                   up.wait_ms, t_setup);
  }
  int fl = 0;
  RK_CUDA(cudaMemcpy(&fl, flag, sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<double> ph(chunk_id * pblocks);
  if (!ph.empty()) RK_CUDA(cudaMemcpy(ph.data(), part, sizeof(double) * ph.size(), cudaMemcpyDeviceToHost));
  dfree(part);
  dfree(flag);
  RK_REQUIRE(!(fl & 1), RK_ERR_DATA, "negative value in tensor");
  RK_REQUIRE(!(fl & 2), RK_ERR_DATA, "column index out of range");
  double s2 = 0.0;
  for (double v : ph) s2 += v;
  const double t_copy = ms_since(t_start);
  auto t_csc = now();
  build_csc(h, bounds);
  h->norm2 = h->norm2_dev = h->norm2_orig = global_sum(h, s2);
  h->have_x = true;
  h->perturbed = false;
  drop_base_copies(h);
  if (timing)
    std::fprintf(stderr, "[rk] upload_csr_slices: copy+validate %.1f ms, csc build %.1f ms (nnz %lld)\n", t_copy,
                 ms_since(t_csc), (long long)nnz);
}
}  // namespace

extern "C" {

int rk_version(void) { return 10000; }

const char* rk_last_error(void) { return g_err.c_str(); }

int rk_device_count(int* out) {
  return guarded([&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *out = n;
  });
}

int rk_create(int device, int64_t n, int64_t m, int32_t k, int32_t engine, rk_handle** out) {
  return guarded([&] {
    RK_REQUIRE(out, RK_ERR_DATA, "null output handle");
    *out = nullptr;
    RK_REQUIRE(n >= 1 && m >= 1, RK_ERR_DATA, "need n >= 1 and m >= 1");
    RK_REQUIRE(1 <= k && k <= n, RK_ERR_DATA,
               "need 1 <= k <= n, got k=" + std::to_string(k) + ", n=" + std::to_string(n));
    RK_REQUIRE(k <= 256, RK_ERR_DATA, "device engine supports k <= 256");
    int ndev = 0;
    RK_CUDA(cudaGetDeviceCount(&ndev));
    RK_REQUIRE(device >= 0 && device < ndev, RK_ERR_DEVICE, "no such CUDA device");
    RK_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    RK_CUDA(cudaGetDeviceProperties(&prop, device));
    RK_REQUIRE(prop.major == 10, RK_ERR_DEVICE,
               std::string("sm_100a build needs a Blackwell (cc 10.x) GPU, found ") + prop.name);
    rk_handle* h = new rk_handle();
    h->dev = device;
    h->num_sms = prop.multiProcessorCount;
    h->n = n;
    h->m = m;
    h->k = k;
    h->K = (int)round_up(k, 16);
    h->requested_engine = engine;
    h->piece = n;
    set_block_dims(h, n, n, round_up(n, 128), round_up(n, 128));
    RK_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    RK_CUDA(cudaMalloc(&h->ctl, sizeof(Ctl)));
    RK_CUDA(cudaMemset(h->ctl, 0, sizeof(Ctl)));
    RK_CUDA(cudaDeviceSynchronize());
    RK_CUDA(cudaMallocHost(&h->ctl_host, sizeof(Ctl)));
    RK_CUDA(cudaMallocHost(&h->stop_host, 2 * sizeof(int)));
    RK_CUDA(cudaEventCreate(&h->ev_run0));
    RK_CUDA(cudaEventCreate(&h->ev_run1));
    h->nnp = h->num_sms * 4;
    h->npart = dalloc<double>(h->nnp);
    h->npart2 = dalloc<double>(h->nnp);
    h->d_iters = dalloc<int>(1);
    alloc_tensor(h);
    alloc_factor_buffers(h);
    *out = h;
  });
}

void rk_destroy(rk_handle* h) {
  if (!h) return;
  cudaSetDevice(h->dev);
  cudaStreamSynchronize(h->stream);
  free_factor_buffers(h);
  dfree(h->Xh);
  dfree(h->Xl);
  dfree(h->Xh0);
  dfree(h->Xl0);
  dfree(h->ctl);
  dfree(h->npart);
  dfree(h->npart2);
  dfree(h->d_iters);
  dfree(h->trace_dev);
  dfree(h->d_colmap);
  void* sps[] = {h->csr_ptr, h->csc_ptr, h->csr_idx, h->csc_idx, h->csr_val, h->csc_val, h->csr_val0,
                 h->csc_val0};
  for (void* p : sps) dfree(p);
  if (h->ctl_host) cudaFreeHost(h->ctl_host);
  if (h->stop_host) cudaFreeHost(h->stop_host);
  for (auto e : h->ev_k1) cudaEventDestroy(e);
  for (auto e : h->ev_ph) cudaEventDestroy(e);
  if (h->ev_run0) cudaEventDestroy(h->ev_run0);
  if (h->ev_run1) cudaEventDestroy(h->ev_run1);
  peer_teardown(h);
  if (h->rowc) ncclCommDestroy(h->rowc);
  if (h->colc) ncclCommDestroy(h->colc);
  if (h->world) ncclCommDestroy(h->world);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

int rk_create_sparse(int device, int64_t n, int64_t m, int32_t k, rk_handle** out) {
  return guarded([&] {
    RK_REQUIRE(out, RK_ERR_DATA, "null output handle");
    *out = nullptr;
    RK_REQUIRE(n >= 1 && m >= 1, RK_ERR_DATA, "need n >= 1 and m >= 1");
    RK_REQUIRE(1 <= k && k <= n, RK_ERR_DATA,
               "need 1 <= k <= n, got k=" + std::to_string(k) + ", n=" + std::to_string(n));
    RK_REQUIRE(k <= 32, RK_ERR_DATA, "sparse engine supports k <= 32");
    RK_REQUIRE(n < (1ll << 31), RK_ERR_DATA, "sparse engine: n must fit int32 indices");
    int ndev = 0;
    RK_CUDA(cudaGetDeviceCount(&ndev));
    RK_REQUIRE(device >= 0 && device < ndev, RK_ERR_DEVICE, "no such CUDA device");
    RK_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    RK_CUDA(cudaGetDeviceProperties(&prop, device));
    RK_REQUIRE(prop.major == 10, RK_ERR_DEVICE,
               std::string("sm_100a build needs a Blackwell (cc 10.x) GPU, found ") + prop.name);
    rk_handle* h = new rk_handle();
    h->sparse = true;
    h->dev = device;
    h->num_sms = prop.multiProcessorCount;
    h->n = n;
    h->m = m;
    h->k = k;
    h->K = k <= 16 ? 16 : 32;
    h->requested_engine = RK_ENGINE_SIMT;
    h->piece = n;
    set_block_dims(h, n, n, round_up(n, 128), round_up(n, 128));
    RK_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    RK_CUDA(cudaMalloc(&h->ctl, sizeof(Ctl)));
    RK_CUDA(cudaMemset(h->ctl, 0, sizeof(Ctl)));
    RK_CUDA(cudaDeviceSynchronize());
    RK_CUDA(cudaMallocHost(&h->ctl_host, sizeof(Ctl)));
    RK_CUDA(cudaMallocHost(&h->stop_host, 2 * sizeof(int)));
    RK_CUDA(cudaEventCreate(&h->ev_run0));
    RK_CUDA(cudaEventCreate(&h->ev_run1));
    h->nnp = h->num_sms * 4;
    h->npart = dalloc<double>(h->nnp);
    h->npart2 = dalloc<double>(h->nnp);
    h->d_iters = dalloc<int>(1);
    alloc_factor_buffers(h);
    *out = h;
  });
}

int rk_upload_csr_slices(rk_handle* h, const int64_t* const* indptrs, const int32_t* const* indices,
                         const void* const* data, const int64_t* nnz_per_slice, int32_t dtype) {
  return guarded([&] {
    RK_REQUIRE(h && h->sparse, RK_ERR_DATA, "rk_upload_csr_slices needs a sparse handle");
    RK_REQUIRE(indptrs && indices && data && nnz_per_slice, RK_ERR_DATA, "null argument");
    RK_CUDA(cudaSetDevice(h->dev));
    upload_csr_slices(h, indptrs, indices, data, nnz_per_slice, dtype);
  });
}

int rk_upload_csr(rk_handle* h, const int64_t* indptr, const int32_t* indices, const void* data,
                  int32_t dtype, int64_t nnz) {
  return guarded([&] {
    RK_REQUIRE(h && h->sparse, RK_ERR_DATA, "rk_upload_csr needs a sparse handle");
    RK_REQUIRE(indptr && (nnz == 0 || (indices && data)), RK_ERR_DATA, "null argument");
    RK_CUDA(cudaSetDevice(h->dev));
    const int64_t rows = h->rows_valid, M = h->m;
    RK_REQUIRE(indptr[0] == 0 && indptr[M * (rows + 1) - 1] == nnz, RK_ERR_DATA, "inconsistent indptr");
    const size_t vsize = dtype == RK_F64 ? 8 : 4;
    std::vector<std::vector<int64_t>> local((size_t)M);
    std::vector<const int64_t*> ip((size_t)M);
    std::vector<const int32_t*> ix((size_t)M);
    std::vector<const void*> dv((size_t)M);
    std::vector<int64_t> cnt((size_t)M);
    for (int64_t t = 0; t < M; ++t) {
      const int64_t* g = indptr + t * (rows + 1);
      const int64_t b0 = g[0];
      local[t].resize((size_t)rows + 1);
      for (int64_t e = 0; e <= rows; ++e) local[t][e] = g[e] - b0;
      ip[t] = local[t].data();
      ix[t] = indices ? indices + b0 : nullptr;
      dv[t] = data ? static_cast<const uint8_t*>(data) + (size_t)b0 * vsize : nullptr;
      cnt[t] = g[rows] - b0;
    }
    upload_csr_slices(h, ip.data(), ix.data(), dv.data(), cnt.data(), dtype);
  });
}

int rk_fill_sparse_uniform(rk_handle* h, uint64_t seed, int64_t nnz_target_per_slice) {
  return guarded([&] {
    RK_REQUIRE(h && h->sparse, RK_ERR_DATA, "needs a sparse handle");
    RK_CUDA(cudaSetDevice(h->dev));
    const int64_t n = h->n, M = h->m, cnt = nnz_target_per_slice;
    const int64_t rows = h->rows_valid, cols = h->cols_valid;
    const int64_t row0 = h->grid() ? (int64_t)h->gi * h->pc * h->piece : 0;
    void* old[] = {h->csr_ptr, h->csc_ptr, h->csr_idx, h->csc_idx, h->csr_val, h->csc_val, h->csr_val0,
                   h->csc_val0};
    for (void* p : old) dfree(p);
    h->csr_val0 = h->csc_val0 = nullptr;
    // a block holds ~ rows*cols/n^2 of the entries; leave slack
    const double frac = h->grid() ? std::min(1.0, 1.25 * (double)rows * cols / ((double)n * n) + 0.01) : 1.0;
    const size_t cap = (size_t)std::ceil((double)M * cnt * frac) + 1024;
    h->csr_ptr = dalloc<int64_t>((size_t)M * (rows + 1));
    h->csc_ptr = dalloc<int64_t>((size_t)M * (cols + 1));
    h->csr_idx = dalloc<int>(cap);
    h->csc_idx = dalloc<int>(cap);
    h->csr_val = dalloc<float>(cap);
    h->csc_val = dalloc<float>(cap);
    int* col_local = nullptr;
    if (h->grid()) {
      std::vector<int> cl((size_t)n, -1);
      for (size_t jl = 0; jl < h->colmap.size(); ++jl)
        if (h->colmap[jl] < n) cl[h->colmap[jl]] = (int)jl;
      col_local = dalloc<int>((size_t)n);
      RK_CUDA(cudaMemcpy(col_local, cl.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
    }
    uint64_t* keys = dalloc<uint64_t>(cnt);
    uint64_t* keys2 = dalloc<uint64_t>(cnt);
    int* flag = dalloc<int>(cnt);
    int* pos = dalloc<int>(cnt);
    int* counts = dalloc<int>(rows);
    size_t t1 = 0, t2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, t1, keys, keys2, (int)cnt, 0, 64, h->stream);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, flag, pos, (int)cnt, h->stream);
    void* tmp = dalloc<uint8_t>(std::max(t1, t2) + 16);
    size_t tmp_bytes = std::max(t1, t2);
    std::vector<int64_t> ptr_host((size_t)M * (rows + 1));
    int64_t base = 0;
    for (int64_t t = 0; t < M; ++t) {
      rk::sp::sp_gen_keys<<<h->num_sms * 8, 256, 0, h->stream>>>(seed, (int)t, cnt, (int)n, keys);
      RK_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, keys2, (int)cnt, 0, 64, h->stream));
      rk::sp::sp_mark_unique_block<<<h->num_sms * 8, 256, 0, h->stream>>>(keys2, cnt, row0, rows, col_local, flag);
      RK_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flag, pos, (int)cnt, h->stream));
      RK_CUDA(cudaMemsetAsync(counts, 0, sizeof(int) * rows, h->stream));
      rk::sp::sp_scatter_unique<<<h->num_sms * 8, 256, 0, h->stream>>>(keys2, flag, pos, cnt, base, h->csr_idx,
                                                                        h->csr_val, counts, seed, (int)t,
                                                                        row0, col_local);
      rk::sp::sp_offsets<<<1, 1024, 0, h->stream>>>(counts, (int)rows, base, h->csr_ptr + t * (rows + 1));
      RK_CUDA(cudaGetLastError());
      RK_CUDA(cudaMemcpyAsync(&ptr_host[t * (rows + 1)], h->csr_ptr + t * (rows + 1),
                              sizeof(int64_t) * (rows + 1), cudaMemcpyDeviceToHost, h->stream));
      RK_CUDA(cudaStreamSynchronize(h->stream));
      base = ptr_host[t * (rows + 1) + rows];
      RK_REQUIRE((size_t)base <= cap, RK_ERR_DEVICE, "sparse generator: block capacity exceeded");
    }
    h->nnz = base;
    dfree(keys);
    dfree(keys2);
    dfree(flag);
    dfree(pos);
    dfree(counts);
    dfree(tmp);
    dfree(col_local);
    std::vector<int64_t> bounds((size_t)M + 1);
    for (int64_t t = 0; t <= M; ++t) bounds[(size_t)t] = t < M ? ptr_host[t * (rows + 1)] : h->nnz;
    build_csc(h, bounds);
    rk::sp::sp_sq_norm<<<h->nnp, 256, 0, h->stream>>>(h->csr_val, h->nnz, h->npart);
    RK_CUDA(cudaStreamSynchronize(h->stream));
    std::vector<double> p(h->nnp);
    RK_CUDA(cudaMemcpy(p.data(), h->npart, sizeof(double) * h->nnp, cudaMemcpyDeviceToHost));
    double s2 = 0.0;
    for (double v : p) s2 += v;
    h->norm2 = h->norm2_dev = h->norm2_orig = global_sum(h, s2);
    h->have_x = true;
    h->perturbed = false;
    drop_base_copies(h);
  });
}

int rk_csr_copy(rk_handle* h, int64_t* indptr, int32_t* indices, float* data) {
  return guarded([&] {
    RK_REQUIRE(h && h->sparse, RK_ERR_DATA, "needs a sparse handle");
    RK_CUDA(cudaSetDevice(h->dev));
    RK_CUDA(cudaMemcpy(indptr, h->csr_ptr, sizeof(int64_t) * h->m * (h->rows_valid + 1), cudaMemcpyDeviceToHost));
    RK_CUDA(cudaMemcpy(indices, h->csr_idx, sizeof(int) * h->nnz, cudaMemcpyDeviceToHost));
    RK_CUDA(cudaMemcpy(data, h->csr_val, sizeof(float) * h->nnz, cudaMemcpyDeviceToHost));
  });
}

int rk_nnz(rk_handle* h, int64_t* out) {
  return guarded([&] { *out = h->nnz; });
}

int rk_csc_copy(rk_handle* h, int64_t* indptr, int32_t* indices, float* data) {
  return guarded([&] {
    RK_REQUIRE(h && h->sparse, RK_ERR_DATA, "needs a sparse handle");
    RK_CUDA(cudaSetDevice(h->dev));
    RK_CUDA(cudaMemcpy(indptr, h->csc_ptr, sizeof(int64_t) * h->m * (h->cols_valid + 1), cudaMemcpyDeviceToHost));
    RK_CUDA(cudaMemcpy(indices, h->csc_idx, sizeof(int) * h->nnz, cudaMemcpyDeviceToHost));
    RK_CUDA(cudaMemcpy(data, h->csc_val, sizeof(float) * h->nnz, cudaMemcpyDeviceToHost));
  });
}

int rk_set_rank(rk_handle* h, int32_t k) {
  return guarded([&] {
    RK_REQUIRE(h, RK_ERR_DATA, "null handle");
    RK_REQUIRE(1 <= k && k <= h->n && k <= 256, RK_ERR_DATA, "bad rank");
    RK_REQUIRE(!h->sparse || k <= 32, RK_ERR_DATA, "sparse engine supports k <= 32");
    RK_CUDA(cudaSetDevice(h->dev));
    RK_CUDA(cudaStreamSynchronize(h->stream));
    free_factor_buffers(h);
    h->k = k;
    h->K = (int)round_up(k, 16);
    alloc_factor_buffers(h);
  });
}

int rk_set_option(rk_handle* h, int32_t key, int64_t value) {
  return guarded([&] {
    RK_REQUIRE(h, RK_ERR_DATA, "null handle");
    if (key == 1) h->profile = value != 0;
    else if (key == 4) h->skip_comm = value != 0;
    else if (key == 2) {
      h->use_graph = value != 0;
      if (!h->use_graph) drop_graphs(h);
    } else
      throw RkError{RK_ERR_DATA, "unknown option"};
  });
}

int rk_upload_dense(rk_handle* h, const void* x, int32_t dtype) {
  return guarded([&] {
    RK_REQUIRE(h && x, RK_ERR_DATA, "null argument");
    RK_REQUIRE(dtype == RK_F32 || dtype == RK_F64, RK_ERR_DATA, "dtype must be f32 or f64");
    RK_REQUIRE(!h->grid(), RK_ERR_GRID, "grid handles take rk_upload_block");
    RK_CUDA(cudaSetDevice(h->dev));
    RK_CUDA(cudaMemsetAsync(h->npart, 0, sizeof(double) * h->nnp, h->stream));
    RK_CUDA(cudaMemsetAsync(h->npart2, 0, sizeof(double) * h->nnp, h->stream));
    if (dtype == RK_F32)
      upload_rows(h, static_cast<const float*>(x), h->n, h->n);
    else
      upload_rows(h, static_cast<const double*>(x), h->n, h->n);
    finish_upload_norm(h, true);
    h->have_x = true;
    h->perturbed = false;
    drop_base_copies(h);
  });
}

int rk_upload_block(rk_handle* h, const void* x, int32_t dtype, int64_t rows, int64_t cols,
                    double sq_norm_global) {
  return guarded([&] {
    RK_REQUIRE(h && x, RK_ERR_DATA, "null argument");
    RK_REQUIRE(rows == h->rows_valid && cols == h->cols_valid, RK_ERR_GRID,
               "block shape does not match the rank's grid block");
    RK_CUDA(cudaSetDevice(h->dev));
    RK_CUDA(cudaMemsetAsync(h->npart, 0, sizeof(double) * h->nnp, h->stream));
    RK_CUDA(cudaMemsetAsync(h->npart2, 0, sizeof(double) * h->nnp, h->stream));
    if (dtype == RK_F32)
      upload_rows(h, static_cast<const float*>(x), rows, cols);
    else
      upload_rows(h, static_cast<const double*>(x), rows, cols);
    // sq_norm_global < 0: the ranks' exact device sums of squares (all-reduced)
    const bool dev_norm = sq_norm_global < 0.0;
    finish_upload_norm(h, dev_norm);
    if (!dev_norm) h->norm2 = sq_norm_global;
    h->have_x = true;
    h->perturbed = false;
    drop_base_copies(h);
  });
}

int rk_fill_uniform(rk_handle* h, uint64_t seed) {
  return guarded([&] {
    RK_REQUIRE(h, RK_ERR_DATA, "null handle");
    RK_CUDA(cudaSetDevice(h->dev));
    rk::fill_uniform<<<h->nnp, rk::kThreads, 0, h->stream>>>(
        h->Xh, h->Xl, h->NR, h->NC, h->rows_valid, h->cols_valid, h->n,
        h->grid() ? (int64_t)h->gi * h->pc * h->piece : 0, h->d_colmap, (int)h->m, seed, h->npart,
        h->npart2);
    RK_CUDA(cudaGetLastError());
    finish_upload_norm(h, true);
    h->have_x = true;
    h->perturbed = false;
    drop_base_copies(h);
  });
}

int rk_uniform_values(uint64_t seed, int64_t offset, int64_t count, float* out) {
  return guarded([&] {
    float* d = dalloc<float>((size_t)count);
    rk::uniform_values<<<1024, 256>>>(d, count, offset, seed);
    RK_CUDA(cudaGetLastError());
    RK_CUDA(cudaMemcpy(out, d, sizeof(float) * count, cudaMemcpyDeviceToHost));
    dfree(d);
  });
}

int rk_block_uniform(rk_handle* h, uint64_t seed, float* out) {
  return guarded([&] {
    RK_REQUIRE(h && out, RK_ERR_DATA, "null argument");
    RK_CUDA(cudaSetDevice(h->dev));
    const size_t count = (size_t)h->m * h->rows_valid * h->cols_valid;
    float* d = dalloc<float>(count);
    rk::block_uniform<<<h->num_sms * 8, rk::kThreads, 0, h->stream>>>(
        d, h->rows_valid, h->cols_valid, h->n, h->grid() ? (int64_t)h->gi * h->pc * h->piece : 0,
        h->d_colmap, (int)h->m, seed);
    RK_CUDA(cudaGetLastError());
    RK_CUDA(cudaMemcpyAsync(out, d, count * sizeof(float), cudaMemcpyDeviceToHost, h->stream));
    RK_CUDA(cudaStreamSynchronize(h->stream));
    dfree(d);
  });
}

int rk_set_factors(rk_handle* h, const double* A, const double* R) {
  return guarded([&] {
    RK_REQUIRE(h && A && R, RK_ERR_DATA, "null argument");
    RK_CUDA(cudaSetDevice(h->dev));
    const int K = h->K, k = h->k;
    std::vector<double> r((size_t)h->m * K * K, 0.0);
    for (int64_t t = 0; t < h->m; ++t)
      for (int a = 0; a < k; ++a)
        for (int b = 0; b < k; ++b) r[((size_t)t * K + a) * K + b] = R[((size_t)t * k + a) * k + b];
    if (!h->grid()) {
      // compact (n, k) straight to the device, padded there to (n, K)
      double* stage = dalloc<double>((size_t)h->n * k);
      RK_CUDA(cudaMemcpyAsync(stage, A, sizeof(double) * h->n * k, cudaMemcpyHostToDevice, h->stream));
      rk::pack_cols<<<h->num_sms * 4, 256, 0, h->stream>>>(stage, h->n, k, h->Arow, K);
      RK_CUDA(cudaGetLastError());
      if (h->NR > h->n)  // padding rows stay exactly zero (rescal.py:144 keeps zeros)
        RK_CUDA(cudaMemsetAsync(h->Arow + (size_t)h->n * K, 0, sizeof(double) * (h->NR - h->n) * K, h->stream));
      RK_CUDA(cudaMemcpyAsync(h->R, r.data(), r.size() * 8, cudaMemcpyHostToDevice, h->stream));
      launch_emit(h);
      RK_CUDA(cudaStreamSynchronize(h->stream));
      dfree(stage);
      return;
    }
    // A: global (n, k) -> this rank's row / col sets, zero padded
    std::vector<double> arow((size_t)h->NR * K, 0.0), acol((size_t)h->NC * K, 0.0);
    const int64_t r0 = h->grid() ? (int64_t)h->gi * h->pc * h->piece : 0;
    for (int64_t i = 0; i < h->rows_valid; ++i) {
      int64_t g = r0 + i;
      if (g < h->n)
        for (int c = 0; c < k; ++c) arow[(size_t)i * K + c] = A[g * k + c];
    }
    if (h->grid())
      for (int64_t j = 0; j < h->cols_valid; ++j) {
        int64_t g = h->colmap[j];
        if (g < h->n)
          for (int c = 0; c < k; ++c) acol[(size_t)j * K + c] = A[g * k + c];
      }
    RK_CUDA(cudaMemcpyAsync(h->Arow, arow.data(), arow.size() * 8, cudaMemcpyHostToDevice, h->stream));
    if (h->grid())
      RK_CUDA(cudaMemcpyAsync(h->Acol, acol.data(), acol.size() * 8, cudaMemcpyHostToDevice, h->stream));
    RK_CUDA(cudaMemcpyAsync(h->R, r.data(), r.size() * 8, cudaMemcpyHostToDevice, h->stream));
    launch_emit(h);
    RK_CUDA(cudaStreamSynchronize(h->stream));
  });
}

int rk_get_factors(rk_handle* h, double* A, double* R) {
  return guarded([&] {
    RK_REQUIRE(h, RK_ERR_DATA, "null handle");
    RK_CUDA(cudaSetDevice(h->dev));
    RK_CUDA(cudaStreamSynchronize(h->stream));
    const int K = h->K, k = h->k;
    if (A) {
      // gather the full A: on a grid every rank's row set covers pc pieces;
      // the (gi, *) row sets tile all n rows, so all-gather row sets over the
      // col communicator.
      std::vector<double> full;
      if (h->grid()) {
        const size_t rs = (size_t)h->pc * h->piece * K;
        double* d = dalloc<double>(rs * h->pr);
        RK_CUDA(cudaMemcpyAsync(d + (size_t)h->gi * rs, h->Arow, rs * 8, cudaMemcpyDeviceToDevice, h->stream));
        RK_NCCL(ncclAllGather(d + (size_t)h->gi * rs, d, rs, ncclDouble, h->colc, h->stream));
        RK_CUDA(cudaStreamSynchronize(h->stream));
        full.resize(rs * h->pr);
        RK_CUDA(cudaMemcpy(full.data(), d, full.size() * 8, cudaMemcpyDeviceToHost));
        dfree(d);
        for (int64_t i = 0; i < h->n; ++i)
          for (int c = 0; c < k; ++c) A[i * k + c] = full[(size_t)i * K + c];
      } else {
        // unpadded on the device, one copy into the caller's (n, k) array
        double* stage = dalloc<double>((size_t)h->n * k);
        rk::unpack_cols<<<h->num_sms * 4, 256, 0, h->stream>>>(h->Arow, K, h->n, k, stage);
        RK_CUDA(cudaGetLastError());
        RK_CUDA(cudaMemcpyAsync(A, stage, sizeof(double) * h->n * k, cudaMemcpyDeviceToHost, h->stream));
        RK_CUDA(cudaStreamSynchronize(h->stream));
        dfree(stage);
      }
    }
    if (R) {
      std::vector<double> r((size_t)h->m * K * K);
      RK_CUDA(cudaMemcpy(r.data(), h->R, r.size() * 8, cudaMemcpyDeviceToHost));
      for (int64_t t = 0; t < h->m; ++t)
        for (int a = 0; a < k; ++a)
          for (int b = 0; b < k; ++b) R[((size_t)t * k + a) * k + b] = r[((size_t)t * K + a) * K + b];
    }
  });
}

int rk_run(rk_handle* h, int32_t iters, double eps, int32_t track_error, double tol,
           double* trace_out, int32_t* iters_done) {
  return guarded([&] {
    check_ready(h);
    RK_REQUIRE(iters >= 1, RK_ERR_DATA, "max_iters must be >= 1");
    if (track_error) RK_REQUIRE(h->norm2 > 0.0, RK_ERR_DATA, "cannot track relative error: tensor norm is zero");
    if (h->eps != eps) drop_graphs(h);
    h->eps = eps;
    ensure_peer(h);
    ensure_trace(h, iters + 1);
    reset_ctl(h, track_error ? 1 : 0, tol, iters);
    h->k1_count = 0;
    h->launches = 0;
    h->ph_iters = 0;
    const bool timed = h->profile;
    // NCCL collectives are stream-capturable: the grid iteration is a graph too
    const bool graph = h->use_graph && !timed;
    const int ti = track_error ? 1 : 0;
    auto get_graph = [&](int batched) {
      cudaGraphExec_t& ge = h->graphs[ti][batched];
      if (!ge) {
        cudaGraph_t g;
        RK_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        const int before = h->launches;
        for (int q = 0; q < (batched ? rk_handle::kGraphBatch : 1); ++q) enqueue_iteration(h, false, ti != 0);
        h->graph_launches[ti][batched] = h->launches - before;
        h->launches = before;  // captured, not launched: counted when the graph runs
        RK_CUDA(cudaStreamEndCapture(h->stream, &g));
        RK_CUDA(cudaGraphInstantiate(&ge, g, 0));
        cudaGraphDestroy(g);
      }
      return ge;
    };
    RK_CUDA(cudaEventRecord(h->ev_run0, h->stream));
    const int chunk = rk_handle::kGraphBatch;
    cudaEvent_t chk[2];
    for (int i = 0; i < 2; ++i) RK_CUDA(cudaEventCreateWithFlags(&chk[i], cudaEventDisableTiming));
    h->launches = 0;
    int launched = 0, pending = -1;
    while (launched < iters) {
      const int nthis = std::min(chunk, iters - launched);
      if (graph && nthis == rk_handle::kGraphBatch) {
        RK_CUDA(cudaGraphLaunch(get_graph(1), h->stream));
        h->launches += h->graph_launches[ti][1];
      } else {
        for (int q = 0; q < nthis; ++q) {
          if (graph) {
            RK_CUDA(cudaGraphLaunch(get_graph(0), h->stream));
            h->launches += h->graph_launches[ti][0];
          } else {
            enqueue_iteration(h, timed, ti != 0);
          }
        }
      }
      launched += nthis;
      const int slot = (launched / chunk) & 1;
      RK_CUDA(cudaMemcpyAsync(&h->stop_host[slot], &h->ctl->stop, sizeof(int), cudaMemcpyDeviceToHost,
                              h->stream));
      RK_CUDA(cudaEventRecord(chk[slot], h->stream));
      if (pending >= 0) {
        RK_CUDA(cudaEventSynchronize(chk[pending]));
        if (h->stop_host[pending]) break;
      }
      pending = slot;
    }
    if (track_error) enqueue_tail(h);
    RK_CUDA(cudaEventRecord(h->ev_run1, h->stream));
    read_ctl(h);
    for (int i = 0; i < 2; ++i) cudaEventDestroy(chk[i]);
    float ms = 0.f;
    RK_CUDA(cudaEventElapsedTime(&ms, h->ev_run0, h->ev_run1));
    h->last_ms = ms;
    for (int p = 0; p < rk_handle::kPhases; ++p) h->ph_ms[p] = 0.0;
    for (int it = 0; it < h->ph_iters; ++it) {
      cudaEvent_t* e = &h->ev_ph[(size_t)it * (rk_handle::kPhases + 1)];
      for (int p = 0; p < rk_handle::kPhases; ++p) {
        // phase 5 exists only on grids; on one GPU phase 4 runs to the end mark
        const int a = p, b = (p == 4 && !h->grid()) ? 6 : p + 1;
        if (p == 5 && !h->grid()) continue;
        float ms = 0.f;
        RK_CUDA(cudaEventElapsedTime(&ms, e[a], e[b == 5 && !h->grid() ? 6 : b]));
        h->ph_ms[p] += ms;
      }
    }
    h->k1_ms_sum = 0.0;
    for (int i = 0; i < h->k1_count; ++i) {
      float e = 0.f;
      RK_CUDA(cudaEventElapsedTime(&e, h->ev_k1[2 * i], h->ev_k1[2 * i + 1]));
      h->k1_ms_sum += e;
    }
    const Ctl& c = *h->ctl_host;
    if (iters_done) *iters_done = c.iter;
    if (track_error && trace_out && c.trace_len > 0)
      RK_CUDA(cudaMemcpy(trace_out, h->trace_dev, sizeof(double) * c.trace_len, cudaMemcpyDeviceToHost));
    if (c.peer_err) throw RkError{RK_ERR_GRID, "peer-memory exchange timed out (a grid rank stopped early)"};
    if (c.nonfinite == 2) throw RkError{RK_ERR_NUMERICAL, "non-finite reconstruction error"};
    if (c.nonfinite) throw RkError{RK_ERR_NUMERICAL, "non-finite value in factors; aborting"};
  });
}

int rk_trace_len(rk_handle* h, int32_t* out) {
  return guarded([&] { *out = h->ctl_host->trace_len; });
}

int rk_update_r(rk_handle* h, double eps) {
  return guarded([&] {
    check_ready(h);
    h->eps = eps;
    reset_ctl(h, 0, -1.0, 1);
    launch_k1(h, false);
    launch_k2a(h, 0);
    if (h->grid()) grid_allreduce_parts(h, false);
    launch_k2f(h, 2);
    read_ctl(h);
    if (h->ctl_host->nonfinite) throw RkError{RK_ERR_NUMERICAL, "non-finite value in factors; aborting"};
  });
}

int rk_update_a(rk_handle* h, double eps) {
  return guarded([&] {
    check_ready(h);
    h->eps = eps;
    reset_ctl(h, 0, -1.0, 1);
    launch_k1(h, false);
    launch_k2a(h, 0);
    if (h->grid()) grid_allreduce_parts(h, false);
    launch_k2f(h, 3);
    launch_k2b(h);
    read_ctl(h);
    if (h->ctl_host->nonfinite) throw RkError{RK_ERR_NUMERICAL, "non-finite value in factors; aborting"};
  });
}

int rk_residual(rk_handle* h, double* sq_residual, double* sq_norm) {
  return guarded([&] {
    check_ready(h);
    reset_ctl(h, 0, -1.0, 0);
    if (h->sparse) {
      // ||X - A R A^T||^2 = ||X||^2 - 2 sum <R_t, A^T X_t A> + sum <R_t, G R_t G>
      launch_k1(h, false);
      launch_k2a(h, 0);
      if (h->grid()) grid_allreduce_parts(h, false);
      launch_k2f(h, 1);
      RK_CUDA(cudaStreamSynchronize(h->stream));
      std::vector<double> tt(2 * h->m);
      RK_CUDA(cudaMemcpy(tt.data(), h->tt, tt.size() * 8, cudaMemcpyDeviceToHost));
      double res = h->norm2;
      for (int64_t t = 0; t < h->m; ++t) res += -2.0 * tt[2 * t] + tt[2 * t + 1];
      if (sq_residual) *sq_residual = std::max(res, 0.0);
      if (sq_norm) *sq_norm = h->norm2;
      return;
    }
    launch_k5(h, 0);
    double* out = h->red;
    rk::sum_scalars<<<1, 256, 0, h->stream>>>(h->rpart, h->nr, out);
    if (h->grid()) RK_NCCL(ncclAllReduce(out, out, 1, ncclDouble, ncclSum, h->world, h->stream));
    RK_CUDA(cudaStreamSynchronize(h->stream));
    double v = 0.0;
    RK_CUDA(cudaMemcpy(&v, out, sizeof(double), cudaMemcpyDeviceToHost));
    if (sq_residual) *sq_residual = v;
    if (sq_norm) *sq_norm = h->norm2;
  });
}

int rk_regress_r(rk_handle* h, int32_t max_iters, double tol, double eps, int32_t* iters_done) {
  return guarded([&] {
    check_ready(h);
    regress_core(h, max_iters, tol, eps, iters_done);
  });
}

int rk_perturb(rk_handle* h, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
               double delta, int64_t n_global, int64_t row0, int64_t col0, const int64_t* col_map) {
  return guarded([&] {
    check_ready(h);
    (void)col0;
    (void)col_map;
    if (h->sparse) {
      if (!h->csr_val0) {
        h->csr_val0 = dalloc<float>(h->nnz);
        h->csc_val0 = dalloc<float>(h->nnz);
        RK_CUDA(cudaMemcpy(h->csr_val0, h->csr_val, h->nnz * 4, cudaMemcpyDeviceToDevice));
        RK_CUDA(cudaMemcpy(h->csc_val0, h->csc_val, h->nnz * 4, cudaMemcpyDeviceToDevice));
        h->norm2_orig = h->norm2;
      }
      rk::u128 st{state_lo, state_hi}, inc{inc_lo, inc_hi};
      const int64_t prow0 = h->grid() ? (int64_t)h->gi * h->pc * h->piece : 0;
      rk::sp::sp_perturb<<<h->num_sms * 8, 256, 0, h->stream>>>(h->csr_ptr, h->csr_idx, h->csr_val0, h->csr_val,
                                                                 (int)h->rows_valid, (int)h->m, 0, st, inc, delta,
                                                                 h->n, prow0, h->d_colmap);
      rk::sp::sp_perturb<<<h->num_sms * 8, 256, 0, h->stream>>>(h->csc_ptr, h->csc_idx, h->csc_val0, h->csc_val,
                                                                 (int)h->cols_valid, (int)h->m, 1, st, inc, delta,
                                                                 h->n, prow0, h->d_colmap);
      RK_CUDA(cudaGetLastError());
      rk::sp::sp_sq_norm<<<h->nnp, 256, 0, h->stream>>>(h->csr_val, h->nnz, h->npart);
      RK_CUDA(cudaStreamSynchronize(h->stream));
      std::vector<double> p(h->nnp);
      RK_CUDA(cudaMemcpy(p.data(), h->npart, sizeof(double) * h->nnp, cudaMemcpyDeviceToHost));
      double s2 = 0.0;
      for (double v : p) s2 += v;
      h->norm2 = h->norm2_dev = global_sum(h, s2);
      h->perturbed = true;
      return;
    }
    if (!h->Xh0) {
      const size_t count = (size_t)h->m * h->NR * h->NC;
      h->Xh0 = dalloc<__nv_bfloat16>(count);
      h->Xl0 = dalloc<__nv_bfloat16>(count);
      RK_CUDA(cudaMemcpyAsync(h->Xh0, h->Xh, count * 2, cudaMemcpyDeviceToDevice, h->stream));
      RK_CUDA(cudaMemcpyAsync(h->Xl0, h->Xl, count * 2, cudaMemcpyDeviceToDevice, h->stream));
      h->norm2_dev0 = h->norm2_dev;
      h->norm2_orig = h->norm2;
    }
    rk::u128 st{state_lo, state_hi}, inc{inc_lo, inc_hi};
    RK_CUDA(cudaMemsetAsync(h->npart2, 0, sizeof(double) * h->nnp, h->stream));
    if (h->d_colmap == nullptr)
      rk::perturb_rows<<<h->nnp, rk::kThreads, 0, h->stream>>>(
          h->Xh0, h->Xl0, h->Xh, h->Xl, h->NR, h->NC, h->rows_valid, h->cols_valid, (int)h->m,
          n_global, row0, st, inc, delta, h->npart);
    else
      rk::perturb_planes<<<h->nnp, rk::kThreads, 0, h->stream>>>(
          h->Xh0, h->Xl0, h->Xh, h->Xl, h->NR, h->NC, h->rows_valid, h->cols_valid, (int)h->m,
          n_global, row0, h->d_colmap, st, inc, delta, 0, h->npart);
    RK_CUDA(cudaGetLastError());
    finish_upload_norm(h, false);
    // the trace denominator of a resampled tensor is its own norm
    h->norm2 = h->norm2_dev;
    h->perturbed = true;
  });
}

int rk_restore(rk_handle* h) {
  return guarded([&] {
    check_ready(h);
    if (h->sparse) {
      if (h->csr_val0) {
        RK_CUDA(cudaMemcpy(h->csr_val, h->csr_val0, h->nnz * 4, cudaMemcpyDeviceToDevice));
        RK_CUDA(cudaMemcpy(h->csc_val, h->csc_val0, h->nnz * 4, cudaMemcpyDeviceToDevice));
        h->norm2 = h->norm2_dev = h->norm2_orig;
      }
      h->perturbed = false;
      return;
    }
    if (h->Xh0) {
      const size_t count = (size_t)h->m * h->NR * h->NC;
      RK_CUDA(cudaMemcpyAsync(h->Xh, h->Xh0, count * 2, cudaMemcpyDeviceToDevice, h->stream));
      RK_CUDA(cudaMemcpyAsync(h->Xl, h->Xl0, count * 2, cudaMemcpyDeviceToDevice, h->stream));
      RK_CUDA(cudaStreamSynchronize(h->stream));
      h->norm2 = h->norm2_orig;
      h->norm2_dev = h->norm2_dev0;
    }
    h->perturbed = false;
  });
}

namespace {
// device buffer freed on every exit path (a throwing launch or copy included)
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { dfree(p); }
};

void pcg64_draws_body(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, uint64_t offset,
                      int64_t count, double* out) {
  RK_REQUIRE(count >= 0 && (count == 0 || out), RK_ERR_DATA, "null argument");
  if (count == 0) return;
  DevBuf d;
  d.p = dalloc<double>((size_t)count);
  rk::u128 st{state_lo, state_hi}, inc{inc_lo, inc_hi};
  const int64_t threads = (count + 63) / 64;
  rk::pcg64_draws<<<(unsigned)((threads + 255) / 256), 256>>>(st, inc, offset, count, static_cast<double*>(d.p));
  RK_CUDA(cudaGetLastError());
  RK_CUDA(cudaMemcpy(out, d.p, sizeof(double) * count, cudaMemcpyDeviceToHost));
}
}  // namespace

int rk_pcg64_draws(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                   uint64_t offset, int64_t count, double* out) {
  return guarded([&] { pcg64_draws_body(state_hi, state_lo, inc_hi, inc_lo, offset, count, out); });
}
int rk_pcg64_draws_on(int32_t device, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                      uint64_t offset, int64_t count, double* out) {
  // runs on `device` and leaves the calling thread's current device as it was
  int prev = -1;
  cudaGetDevice(&prev);
  const int rc = guarded([&] {
    RK_CUDA(cudaSetDevice(device));
    pcg64_draws_body(state_hi, state_lo, inc_hi, inc_lo, offset, count, out);
  });
  if (prev >= 0) cudaSetDevice(prev);
  return rc;
}
int rk_perturb_values(int32_t device, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                      double delta, int32_t dtype, void* values, int64_t count, uint64_t e0, int32_t field_only) {
  return guarded([&] {
    RK_REQUIRE(dtype == RK_F32 || dtype == RK_F64, RK_ERR_DATA, "unsupported dtype");
    RK_REQUIRE(count >= 0 && (count == 0 || values), RK_ERR_DATA, "null argument");
    RK_CUDA(cudaSetDevice(device));
    if (count == 0) return;
    const rk::u128 st{state_lo, state_hi}, inc{inc_lo, inc_hi};
    const size_t esz = dtype == RK_F32 ? 4 : 8;
    // chunks of whole 2048-element segments so every chunk restarts cleanly
    const int64_t chunk = (int64_t)((256ull << 20) / esz);
    uint8_t* d = dalloc<uint8_t>((size_t)std::min<int64_t>(count, chunk) * esz);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    for (int64_t o = 0; o < count; o += chunk) {
      const int64_t c = std::min(chunk, count - o);
      uint8_t* hv = static_cast<uint8_t*>(values) + (size_t)o * esz;
      if (!field_only) RK_CUDA(cudaMemcpy(d, hv, (size_t)c * esz, cudaMemcpyHostToDevice));
      if (dtype == RK_F32)
        rk::perturb_flat<float><<<sms * 8, 256>>>(reinterpret_cast<float*>(d), c, e0 + (uint64_t)o, st, inc, delta,
                                                  field_only);
      else
        rk::perturb_flat<double><<<sms * 8, 256>>>(reinterpret_cast<double*>(d), c, e0 + (uint64_t)o, st, inc,
                                                   delta, field_only);
      RK_CUDA(cudaGetLastError());
      RK_CUDA(cudaMemcpy(hv, d, (size_t)c * esz, cudaMemcpyDeviceToHost));
    }
    dfree(d);
  });
}

int rk_perturb_csr_values(int32_t device, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                          double delta, int32_t dtype, int64_t t, int64_t n, const int64_t* indptr,
                          const int32_t* indices, void* values, int64_t nnz) {
  return guarded([&] {
    RK_REQUIRE(dtype == RK_F32 || dtype == RK_F64, RK_ERR_DATA, "unsupported dtype");
    RK_REQUIRE(indptr && (nnz == 0 || (indices && values)), RK_ERR_DATA, "null argument");
    RK_REQUIRE(indptr[0] == 0 && indptr[n] == nnz, RK_ERR_DATA, "inconsistent indptr");
    RK_CUDA(cudaSetDevice(device));
    if (nnz == 0) return;
    const rk::u128 st{state_lo, state_hi}, inc{inc_lo, inc_hi};
    const size_t esz = dtype == RK_F32 ? 4 : 8;
    int64_t* dp = dalloc<int64_t>((size_t)n + 1);
    int* di = dalloc<int>((size_t)nnz);
    uint8_t* dv = dalloc<uint8_t>((size_t)nnz * esz);
    RK_CUDA(cudaMemcpy(dp, indptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
    RK_CUDA(cudaMemcpy(di, indices, sizeof(int) * nnz, cudaMemcpyHostToDevice));
    RK_CUDA(cudaMemcpy(dv, values, esz * nnz, cudaMemcpyHostToDevice));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (dtype == RK_F32)
      rk::perturb_csr_vals<float><<<sms * 8, 256>>>(reinterpret_cast<float*>(dv), dp, di, n, t, n, st, inc, delta);
    else
      rk::perturb_csr_vals<double><<<sms * 8, 256>>>(reinterpret_cast<double*>(dv), dp, di, n, t, n, st, inc, delta);
    RK_CUDA(cudaGetLastError());
    RK_CUDA(cudaMemcpy(values, dv, esz * nnz, cudaMemcpyDeviceToHost));
    dfree(dp);
    dfree(di);
    dfree(dv);
  });
}

// ---- NNDSVD support (rescal.py:327-372): products with the unfolding
// M = [X_1 .. X_m | X_1^T .. X_m^T] for the device subspace iteration.
namespace {
struct UnfoldBufs {
  float *V = nullptr, *P1 = nullptr, *Q1 = nullptr;
  ~UnfoldBufs() {
    dfree(V);
    dfree(P1);
    dfree(Q1);
  }
};

void check_unfold(rk_handle* h, int b) {
  RK_REQUIRE(h != nullptr, RK_ERR_DATA, "null handle");
  RK_REQUIRE(h->have_x, RK_ERR_DATA, "no tensor uploaded");
  RK_REQUIRE(!h->grid(), RK_ERR_GRID, "unfolding products run on a single-GPU handle");
  if (h->sparse)
    RK_REQUIRE(b == 16 || b == 32, RK_ERR_DATA, "sparse unfolding products need a block width of 16 or 32");
  else
    RK_REQUIRE(b >= 1 && b <= 256, RK_ERR_DATA, "dense unfolding products need 1 <= block width <= 256");
  RK_CUDA(cudaSetDevice(h->dev));
}

// out_p[t] = X_t B(t), out_q[t] = X_t^T B'(t); B(t) = V + t*sv, B'(t) = W + t*sw
void unfold_products(rk_handle* h, int b, const float* V, int64_t sv, const float* W, int64_t sw, float* out_p,
                     float* out_q) {
  const int M = (int)h->m;
  if (h->sparse) {
    const int grid = h->num_sms * 16;
    if (b == 16) {
      rk::sp::sp_csr_pass<16><<<grid, 256, 0, h->stream>>>(h->ctl, h->csr_ptr, h->csr_idx, h->csr_val, V, out_p,
                                                          (int)h->rows_valid, (int)h->NR, M, 0, sv);
      rk::sp::sp_csr_pass<16><<<grid, 256, 0, h->stream>>>(h->ctl, h->csc_ptr, h->csc_idx, h->csc_val, W, out_q,
                                                          (int)h->cols_valid, (int)h->NC, M, 0, sw);
    } else {
      rk::sp::sp_csr_pass<32><<<grid, 256, 0, h->stream>>>(h->ctl, h->csr_ptr, h->csr_idx, h->csr_val, V, out_p,
                                                          (int)h->rows_valid, (int)h->NR, M, 0, sv);
      rk::sp::sp_csr_pass<32><<<grid, 256, 0, h->stream>>>(h->ctl, h->csc_ptr, h->csc_idx, h->csc_val, W, out_q,
                                                          (int)h->cols_valid, (int)h->NC, M, 0, sw);
    }
  } else {
    const size_t smem = (size_t)(64 * 33 + 64 * b) * sizeof(float);
    RK_CUDA(cudaFuncSetAttribute(rk::k1_simt_p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    RK_CUDA(cudaFuncSetAttribute(rk::k1_simt_q, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    rk::k1_simt_p<<<dim3((unsigned)(h->NR / 32), M), rk::kThreads, smem, h->stream>>>(
        h->ctl, h->Xh, h->Xl, V, out_p, (int)h->NR, (int)h->NC, b, 0, sv);
    rk::k1_simt_q<<<dim3((unsigned)(h->NC / 32), M), rk::kThreads, smem, h->stream>>>(
        h->ctl, h->Xh, h->Xl, W, out_q, (int)h->NR, (int)h->NC, b, 0, sw);
  }
  RK_CUDA(cudaGetLastError());
}

float* upload_block_cols(rk_handle* h, const double* V, int b) {
  const int64_t n = h->n, ld = std::max(h->NR, h->NC);
  std::vector<float> v32((size_t)ld * b, 0.f);
  for (int64_t e = 0; e < n * b; ++e) v32[e] = (float)V[e];
  float* d = dalloc<float>(v32.size());
  RK_CUDA(cudaMemcpy(d, v32.data(), sizeof(float) * v32.size(), cudaMemcpyHostToDevice));
  return d;
}
}  // namespace

int rk_gram_apply(rk_handle* h, const double* V, int32_t b, double* Y) {
  return guarded([&] {
    check_unfold(h, b);
    RK_REQUIRE(V && Y, RK_ERR_DATA, "null argument");
    const int64_t M = h->m, n = h->n, ld = std::max(h->NR, h->NC);
    UnfoldBufs u;
    u.V = upload_block_cols(h, V, b);
    u.P1 = dalloc<float>((size_t)M * ld * b);
    u.Q1 = dalloc<float>((size_t)M * ld * b);
    float* P2 = dalloc<float>((size_t)M * ld * b);
    float* Q2 = dalloc<float>((size_t)M * ld * b);
    double* Yd = dalloc<double>((size_t)n * b);
    unfold_products(h, b, u.V, 0, u.V, 0, u.P1, u.Q1);                      // X_t V, X_t^T V
    unfold_products(h, b, u.Q1, ld * b, u.P1, ld * b, P2, Q2);             // X_t (X_t^T V), X_t^T (X_t V)
    rk::sum_slices<<<h->num_sms * 4, 256, 0, h->stream>>>(P2, Q2, (int)M, n, ld, b, Yd);
    RK_CUDA(cudaGetLastError());
    RK_CUDA(cudaStreamSynchronize(h->stream));
    RK_CUDA(cudaMemcpy(Y, Yd, sizeof(double) * n * b, cudaMemcpyDeviceToHost));
    dfree(P2);
    dfree(Q2);
    dfree(Yd);
  });
}

int rk_unfold_sign_norms(rk_handle* h, const double* U, int32_t b, double* pos2, double* neg2) {
  return guarded([&] {
    check_unfold(h, b);
    RK_REQUIRE(U && pos2 && neg2, RK_ERR_DATA, "null argument");
    const int64_t M = h->m, n = h->n, ld = std::max(h->NR, h->NC);
    UnfoldBufs u;
    u.V = upload_block_cols(h, U, b);
    u.P1 = dalloc<float>((size_t)M * ld * b);
    u.Q1 = dalloc<float>((size_t)M * ld * b);
    unfold_products(h, b, u.V, 0, u.V, 0, u.P1, u.Q1);
    const int nblk = h->num_sms;
    double* part = dalloc<double>((size_t)nblk * 2 * b);
    rk::sign_norms<<<dim3(nblk, b), 256, 256 * 2 * sizeof(double), h->stream>>>(u.P1, u.Q1, (int)M, n, ld, b, part);
    RK_CUDA(cudaGetLastError());
    std::vector<double> ph((size_t)nblk * 2 * b);
    RK_CUDA(cudaStreamSynchronize(h->stream));
    RK_CUDA(cudaMemcpy(ph.data(), part, sizeof(double) * ph.size(), cudaMemcpyDeviceToHost));
    dfree(part);
    for (int c = 0; c < b; ++c) {
      double a = 0.0, z = 0.0;
      for (int k = 0; k < nblk; ++k) {
        a += ph[(size_t)k * 2 * b + c];
        z += ph[(size_t)k * 2 * b + b + c];
      }
      pos2[c] = a;
      neg2[c] = z;
    }
  });
}

int rk_positive_mean(rk_handle* h, double* mean) {
  return guarded([&] {
    RK_REQUIRE(h && mean, RK_ERR_DATA, "null argument");
    RK_REQUIRE(h->have_x, RK_ERR_DATA, "no tensor uploaded");
    RK_CUDA(cudaSetDevice(h->dev));
    const int nblk = h->num_sms * 2;
    double* part = dalloc<double>((size_t)nblk * 2);
    if (h->sparse)
      rk::positive_sum_flat<<<nblk, 256, 0, h->stream>>>(h->csr_val, h->nnz, part);
    else
      rk::positive_sum<<<nblk, 256, 0, h->stream>>>(h->Xh, h->Xl, (int)h->m, h->NR, h->NC, h->rows_valid,
                                                     h->cols_valid, part);
    RK_CUDA(cudaGetLastError());
    std::vector<double> ph((size_t)nblk * 2);
    RK_CUDA(cudaStreamSynchronize(h->stream));
    RK_CUDA(cudaMemcpy(ph.data(), part, sizeof(double) * ph.size(), cudaMemcpyDeviceToHost));
    dfree(part);
    double s = 0.0, c = 0.0;
    for (int k = 0; k < nblk; ++k) {
      s += ph[2 * k];
      c += ph[2 * k + 1];
    }
    *mean = c > 0 ? s / c : 0.0;
  });
}

void rk_release_cached_memory(void) { pool_release(-1); }

int rk_debug_guards(int32_t on) {
  return guarded([&] {
    pool_release(-1);  // later allocations come fresh (guarded or pooled)
    DevPool& P = dev_pool();
    std::lock_guard<std::mutex> lk(P.mu);
    P.guard = on != 0;
  });
}

int rk_debug_read_pq(rk_handle* h, float* P, float* Q) {
  return guarded([&] {
    RK_REQUIRE(h && h->P && h->Q && h->NR == h->NC, RK_ERR_DATA, "no dense K1 products on this handle");
    RK_CUDA(cudaStreamSynchronize(h->stream));
    RK_CUDA(cudaMemcpy(P, h->P, sizeof(float) * h->m * h->NR * h->K, cudaMemcpyDeviceToHost));
    RK_CUDA(cudaMemcpy(Q, h->Q, sizeof(float) * h->m * h->NC * h->K, cudaMemcpyDeviceToHost));
  });
}

// positive control for the guard check: a 1000-byte block, then `nbytes`
// bytes written right after its end (a deliberate overrun), then freed
int rk_debug_overrun(int64_t nbytes) {
  return guarded([&] {
    RK_REQUIRE(nbytes >= 0 && nbytes <= (int64_t)kGuard, RK_ERR_DATA, "bad overrun size");
    unsigned char* p = dalloc<unsigned char>(1000);
    if (nbytes) RK_CUDA(cudaMemset(p + 1000, 0, (size_t)nbytes));
    RK_CUDA(cudaDeviceSynchronize());
    dfree(p);
  });
}

int rk_debug_check_guards(int64_t* damaged_bytes, int64_t* blocks_checked) {
  return guarded([&] {
    DevPool& P = dev_pool();
    std::lock_guard<std::mutex> lk(P.mu);
    int64_t bad = P.violations;
    for (auto& kv : P.guarded) bad += guard_damage(kv.first, kv.second, P.live[kv.first].first);
    if (damaged_bytes) *damaged_bytes = bad;
    if (blocks_checked) *blocks_checked = (int64_t)P.guarded.size();
  });
}

int rk_nccl_unique_id(void* out128) {
  return guarded([&] {
    ncclUniqueId id;
    RK_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
  });
}

int rk_grid_init(rk_handle* h, int32_t pr, int32_t pc, int32_t rank, const void* nccl_id,
                 int64_t n_global) {
  return guarded([&] {
    RK_REQUIRE(h && nccl_id, RK_ERR_DATA, "null argument");
    RK_REQUIRE(pr >= 1 && pc >= 1 && rank >= 0 && rank < pr * pc, RK_ERR_GRID, "bad grid shape");
    RK_REQUIRE(n_global == h->n, RK_ERR_GRID, "n mismatch");
    RK_CUDA(cudaSetDevice(h->dev));
    RK_CUDA(cudaStreamSynchronize(h->stream));
    const int p = pr * pc;
    h->pr = pr;
    h->pc = pc;
    h->rank = rank;
    h->gi = rank / pc;
    h->gj = rank % pc;
    h->piece = (h->n + p - 1) / p;
    const int64_t b = h->piece;
    set_block_dims(h, pc * b, pr * b, round_up(pc * b, 128), round_up(pr * b, 128));
    h->colmap.resize(pr * b);
    for (int ip = 0; ip < pr; ++ip)
      for (int64_t r = 0; r < b; ++r) h->colmap[ip * b + r] = ((int64_t)ip * pc + h->gj) * b + r;
    dfree(h->d_colmap);
    h->d_colmap = dalloc<int64_t>(h->colmap.size());
    RK_CUDA(cudaMemcpy(h->d_colmap, h->colmap.data(), h->colmap.size() * 8, cudaMemcpyHostToDevice));
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    if (p > 1) {
      RK_NCCL(ncclCommInitRank(&h->world, p, id, rank));
      RK_NCCL(ncclCommSplit(h->world, h->gi, h->gj, &h->rowc, nullptr));
      RK_NCCL(ncclCommSplit(h->world, h->gj, h->gi, &h->colc, nullptr));
    }
    free_factor_buffers(h);
    alloc_tensor(h);
    alloc_factor_buffers(h);
    h->have_x = false;
  });
}

// RESCALk replicas: rank 0 exports its uploaded tensor planes through CUDA
// IPC; the other ranks copy them peer-to-peer over NVLink.
struct TensorExport {
  cudaIpcMemHandle_t xh, xl;
  double norm2, norm2_dev;
  int64_t m, NR, NC;
};

int rk_tensor_export(rk_handle* h, void* out, int32_t out_bytes) {
  return guarded([&] {
    RK_REQUIRE(h && out && out_bytes >= (int32_t)sizeof(TensorExport), RK_ERR_DATA, "bad argument");
    RK_REQUIRE(!h->sparse && !h->grid() && h->have_x && !h->perturbed, RK_ERR_DATA,
               "export needs an uploaded, unperturbed dense single-GPU tensor");
    RK_CUDA(cudaSetDevice(h->dev));
    RK_CUDA(cudaStreamSynchronize(h->stream));
    TensorExport e{};
    RK_CUDA(cudaIpcGetMemHandle(&e.xh, h->Xh));
    RK_CUDA(cudaIpcGetMemHandle(&e.xl, h->Xl));
    e.norm2 = h->norm2;
    e.norm2_dev = h->norm2_dev;
    e.m = h->m;
    e.NR = h->NR;
    e.NC = h->NC;
    std::memcpy(out, &e, sizeof(e));
  });
}

int rk_tensor_import(rk_handle* h, const void* in) {
  return guarded([&] {
    RK_REQUIRE(h && in, RK_ERR_DATA, "null argument");
    TensorExport e;
    std::memcpy(&e, in, sizeof(e));
    RK_REQUIRE(!h->sparse && !h->grid() && e.m == h->m && e.NR == h->NR && e.NC == h->NC, RK_ERR_DATA,
               "exported tensor does not match this handle");
    RK_CUDA(cudaSetDevice(h->dev));
    void *ph = nullptr, *pl = nullptr;
    RK_CUDA(cudaIpcOpenMemHandle(&ph, e.xh, cudaIpcMemLazyEnablePeerAccess));
    cudaError_t err = cudaIpcOpenMemHandle(&pl, e.xl, cudaIpcMemLazyEnablePeerAccess);
    if (err != cudaSuccess) {
      cudaIpcCloseMemHandle(ph);
      RK_CUDA(err);
    }
    const size_t bytes = (size_t)h->m * h->NR * h->NC * sizeof(__nv_bfloat16);
    RK_CUDA(cudaMemcpyAsync(h->Xh, ph, bytes, cudaMemcpyDeviceToDevice, h->stream));
    RK_CUDA(cudaMemcpyAsync(h->Xl, pl, bytes, cudaMemcpyDeviceToDevice, h->stream));
    RK_CUDA(cudaStreamSynchronize(h->stream));
    cudaIpcCloseMemHandle(ph);
    cudaIpcCloseMemHandle(pl);
    h->norm2 = e.norm2;
    h->norm2_dev = h->norm2_dev0 = e.norm2_dev;
    h->have_x = true;
    h->perturbed = false;
    drop_base_copies(h);
  });
}

int rk_grid_block(rk_handle* h, int64_t* out, int32_t n_out) {
  return guarded([&] {
    int64_t v[8] = {h->gi, h->gj, h->piece, h->rows_valid, h->cols_valid,
                    h->grid() ? (int64_t)h->gi * h->pc * h->piece : 0, h->pr, h->pc};
    for (int i = 0; i < n_out && i < 8; ++i) out[i] = v[i];
  });
}

int rk_grid_colmap(rk_handle* h, int64_t* out) {
  return guarded([&] {
    for (size_t i = 0; i < h->colmap.size(); ++i) out[i] = h->colmap[i];
  });
}

int rk_last_timing(rk_handle* h, double* out, int32_t n_out) {
  return guarded([&] {
    double v[4] = {h->last_ms, h->k1_count ? h->k1_ms_sum / h->k1_count : 0.0, (double)h->k1_count,
                   (double)h->launches};
    for (int i = 0; i < n_out && i < 4; ++i) out[i] = v[i];
  });
}

int rk_phase_timing(rk_handle* h, double* out, int32_t n_out) {
  return guarded([&] {
    for (int p = 0; p < n_out && p < rk_handle::kPhases; ++p)
      out[p] = h->ph_iters ? h->ph_ms[p] / h->ph_iters : 0.0;
  });
}

int rk_time_k1(rk_handle* h, int32_t reps, double* ms_per_launch) {
  return guarded([&] {
    check_ready(h);
    reset_ctl(h, 0, -1.0, 0);
    cudaEvent_t a, b;
    RK_CUDA(cudaEventCreate(&a));
    RK_CUDA(cudaEventCreate(&b));
    launch_k1(h, false);
    RK_CUDA(cudaEventRecord(a, h->stream));
    for (int i = 0; i < reps; ++i) launch_k1(h, false);
    RK_CUDA(cudaEventRecord(b, h->stream));
    RK_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    RK_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *ms_per_launch = ms / reps;
  });
}

void* rk_stream(rk_handle* h) { return h ? (void*)h->stream : nullptr; }

int rk_info(rk_handle* h, int64_t* out, int32_t n_out) {
  return guarded([&] {
    RK_REQUIRE(h, RK_ERR_DATA, "null handle");
    int64_t v[14] = {h->engine, h->NR, h->K, h->c, h->grid_tc, (int64_t)h->smem_tc,
                     h->nstrips, h->nslots, h->nb, h->NC, h->peer ? 1 : 0, h->k1_mq ? 1 : 0,
                     h->k1_grp, h->sw};
    for (int i = 0; i < n_out && i < 14; ++i) out[i] = v[i];
  });
}

}  // extern "C"
