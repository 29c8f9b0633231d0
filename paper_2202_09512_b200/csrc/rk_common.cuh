// Shared device helpers for the RESCAL MU engine (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define RK_DEV __device__ __forceinline__

namespace rk {

// Device-side run control. One instance per handle, in device memory; every
// per-iteration kernel reads it so that a stop (tolerance reached, non-finite
// factors) turns the rest of an already-enqueued batch into no-ops without a
// host round trip.
struct Ctl {
  int stop;        // 1: tolerance reached or fatal flag; later kernels no-op
  int direct;      // 1: trace uses the direct residual pass (small errors)
  int nonfinite;   // 1: a non-finite factor value was produced
  int iter;        // iterations committed in the current run
  int trace_len;   // trace entries written in the current run
  int track;       // track_error
  int tail;        // 1: trace-only pass (no factor updates)
  int max_iters;
  double tol;        // < 0: none
  double eps;        // cast to the tensor dtype by the caller
  double norm2;      // ||X||^2 from the host values (fp64) — trace denominator
  double norm2_dev;  // sum (hi+lo)^2 of the device tensor — identity residual
  double direct_thresh;  // switch to the direct residual below this error
  double last_err;
  int peer_err;      // 1: a peer-memory exchange timed out (grid; see peer.cuh)
  int pad_i;
  double pad[5];
};

// Programmatic dependent launch: let the next kernel of the stream be
// scheduled now (its CTAs wait in their own pdl_entry), then wait until every
// kernel this one depends on has completed and its writes are visible. A no-op
// pair for kernels launched without the PDL attribute.
RK_DEV void pdl_entry() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// sum_{c < nchunk} p[c * stride], added in chunk order; the loads go out
// eight at a time (independent, in flight together) instead of one chained
// L2 round trip per chunk (cfg3: 64 chunks).
RK_DEV double sum_chunks(const double* __restrict__ p, int nchunk, int stride) {
  double v = 0.0;
  int c = 0;
  for (; c + 8 <= nchunk; c += 8) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldcg(p + (size_t)(c + u) * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) v += x[u];
  }
  for (; c < nchunk; ++c) v += __ldcg(p + (size_t)c * stride);
  return v;
}

// sum_chunks for NG elements at once (p[i], valid[i]): the same per-element
// order (bit-identical), with the 8-chunk batches of all NG elements in
// flight together (latency-bound reductions: NG x more loads per round trip).
template <int NG>
RK_DEV void sum_chunks_group(const double* const (&p)[NG], const bool (&valid)[NG], int nchunk, int stride,
                             double (&out)[NG]) {
#pragma unroll
  for (int i = 0; i < NG; ++i) out[i] = 0.0;
  int c = 0;
  for (; c + 8 <= nchunk; c += 8) {
    double x[NG][8];
#pragma unroll
    for (int i = 0; i < NG; ++i)
#pragma unroll
      for (int u = 0; u < 8; ++u) x[i][u] = valid[i] ? __ldcg(p[i] + (size_t)(c + u) * stride) : 0.0;
#pragma unroll
    for (int i = 0; i < NG; ++i)
#pragma unroll
      for (int u = 0; u < 8; ++u) out[i] += x[i][u];
  }
  for (; c < nchunk; ++c)
#pragma unroll
    for (int i = 0; i < NG; ++i)
      if (valid[i]) out[i] += __ldcg(p[i] + (size_t)c * stride);
}

RK_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

RK_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Split a value into bf16 hi + bf16 lo with hi = rn(x), lo = rn(x - hi):
// hi + lo carries ~17 significant bits (relative error <= 2^-18).
RK_DEV void split_bf16(double x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __double2bfloat16(x);
  lo = __double2bfloat16(x - (double)__bfloat162float(hi));
}

RK_DEV float join_bf16(__nv_bfloat16 hi, __nv_bfloat16 lo) {
  return __bfloat162float(hi) + __bfloat162float(lo);
}

// Counter-based uniform [0,1) in fp32 (synthetic benchmark inputs only).
RK_DEV uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

RK_DEV float uniform01_f32(uint64_t seed, uint64_t idx) {
  uint64_t r = splitmix64(seed * 0x632BE59BD9B4E019ull + idx);
  return (float)(r >> 40) * (1.0f / 16777216.0f);
}

}  // namespace rk
