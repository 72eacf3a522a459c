// Small device helpers shared by the two tcgen05 scoring kernels (score_tc.cu: resident operand
// image; score_tcs.cu: streamed operands).
#pragma once
#include <cstdint>

#include "gpbo_internal.cuh"
#include <cuda_fp16.h>

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

// Candidate loader, rows with d % 4 == 0 (16-byte aligned rows in the staging buffer): converts
// raw row r into the float16 hi/lo augmented A operand [x^, |x^|^2, 1, 0 ...] of kb 16-wide K
// blocks (SWIZZLE_32B K-major at a0) with float4 shared-memory loads (a warp's 16-byte row loads
// at stride 4 d floats are bank-conflict free; the scalar path's stride-d loads are 4-way
// conflicted at d = 20) and no per-element range branches.  Returns |x^|^2 and the NaN flag.
__device__ __forceinline__ void convert_row_vec4(const float *stg, const float *w, int r, int d,
                                                 int kb, bool valid, uint32_t a0, float &qh_out,
                                                 bool &nan_out) {
  const float4 *x4 = reinterpret_cast<const float4 *>(stg + r * d);
  const float4 *w4 = reinterpret_cast<const float4 *>(w);
  const int d4 = d >> 2;
  float qa = 0.f, qb = 0.f;
  bool nan = false;
  if (valid)
    for (int c = 0; c < d4; ++c) {
      const float4 a = x4[c], ww = w4[c];
      nan |= !(isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(a.w));
      const float v0 = a.x * ww.x, v1 = a.y * ww.y, v2 = a.z * ww.z, v3 = a.w * ww.w;
      qa = fmaf(v0, v0, qa);
      qb = fmaf(v1, v1, qb);
      qa = fmaf(v2, v2, qa);
      qb = fmaf(v3, v3, qb);
    }
  const float qh = qa + qb;
  const bool on = valid && qh <= 30000.f;
  for (int k = 0; k < kb; ++k) {
    uint32_t hw[8], lw[8];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const int c0 = 16 * k + 4 * g;
      float v[4];
      if (on && c0 + 4 <= d) {
        const float4 a = x4[c0 >> 2], ww = w4[c0 >> 2];
        v[0] = a.x * ww.x; v[1] = a.y * ww.y; v[2] = a.z * ww.z; v[3] = a.w * ww.w;
      } else {  // c0 >= d (d % 4 == 0): the augmented columns and zero padding
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = !on ? 0.f : (c0 + u == d ? qh : (c0 + u == d + 1 ? 1.f : 0.f));
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const __half2 h2 = __floats2half2_rn(v[2 * h], v[2 * h + 1]);
        const float2 hf = __half22float2(h2);
        hw[2 * g + h] = *reinterpret_cast<const uint32_t *>(&h2);
        lw[2 * g + h] = tc::pack_f16x2(v[2 * h] - hf.x, v[2 * h + 1] - hf.y);
      }
    }
    const uint32_t base = a0 + k * 8192;
    sts128(base + tc::sw_offset(r, 0, 32), hw[0], hw[1], hw[2], hw[3]);
    sts128(base + tc::sw_offset(r, 16, 32), hw[4], hw[5], hw[6], hw[7]);
    sts128(base + 4096 + tc::sw_offset(r, 0, 32), lw[0], lw[1], lw[2], lw[3]);
    sts128(base + 4096 + tc::sw_offset(r, 16, 32), lw[4], lw[5], lw[6], lw[7]);
  }
  qh_out = qh;
  nan_out = nan;
}

}  // namespace gpbo
