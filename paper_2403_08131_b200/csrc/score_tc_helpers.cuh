// Small device helpers shared by the two tcgen05 scoring kernels (score_tc.cu: resident operand
// image; score_tcs.cu: streamed operands).
#pragma once
#include <cstdint>

#include "gpbo_internal.cuh"
#include "tc_prims.cuh"

namespace gpbo {

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                       uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

__device__ __forceinline__ int search_of(const int32_t *tile_first, int S, int t) {
  int lo = 0, hi = S;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (tile_first[mid] <= t) lo = mid; else hi = mid;
  }
  return lo;
}

// optional event trace of CTA 0 (gpbo_debug_trace): each recording thread owns a slice of
// 16384 entries (fire-and-forget stores, no atomics): slot = role slice + 2 * local count
__device__ __forceinline__ void trace_ev(unsigned long long *tr, uint32_t tag, uint32_t role,
                                         uint32_t idx, uint32_t &cnt) {
#ifndef GPBO_TC_TRACE
  return;  // compiled out unless built with -DGPBO_TC_TRACE (tools/trace_tc.py)
#endif
  if (tr == nullptr || blockIdx.x != 0) return;
  const unsigned long long c = clock64();
  const uint32_t slice = role == 11 ? 0u : role == 8 ? 1u : role == 0 ? 2u : role == 9 ? 4u : 3u;
  if (2 * cnt + 2 < 16384) {
    unsigned long long *b = tr + slice * 16384;
    b[2 * cnt] = ((unsigned long long)tag << 56) | ((unsigned long long)role << 48) | idx;
    b[2 * cnt + 1] = c;
  }
  ++cnt;
}

}  // namespace gpbo
