// Device helpers shared by the scoring kernels: kernel values, EI, key packing, argmax.
#pragma once
#include <cstdint>

#include "gpbo_internal.cuh"

namespace gpbo {



// k(r) in float32 (reading R1/R2): RBF sf2 exp(-r^2/2); Matern-5/2 sf2 (1 + s + s^2/3) e^-s,
// s = sqrt(5) r.
__device__ __forceinline__ float kernel_f32(float r2, float sf2, int kind) {
  if (kind == GPBO_RBF) return sf2 * expf(-0.5f * r2);
  const float sr = sqrtf(5.f * r2);
  return sf2 * fmaf(sr, fmaf(sr, 1.f / 3.f, 1.f), 1.f) * expf(-sr);
}

// tau(z) = phi(z) + z Phi(z).  For z < 0 the direct form cancels; use
// tau(-x) = e^{-x^2/2} [1/sqrt(2 pi) - (x/2) erfcx(x/sqrt 2)].
__device__ __forceinline__ float tau_f32(float z) {
  const float inv_sqrt2pi = 0.398942280401432678f;
  const float inv_sqrt2 = 0.707106781186547524f;
  if (z >= 0.f) return fmaf(z, 0.5f * erfcf(-z * inv_sqrt2), inv_sqrt2pi * expf(-0.5f * z * z));
  const float x = -z;
  return expf(-0.5f * z * z) * fmaf(-0.5f * x, erfcxf(x * inv_sqrt2), inv_sqrt2pi);
}

// EI for minimisation (readings R3, R4): s tau((best - mu)/s), or
// max(best - mu, 0) when s == 0.
__device__ __forceinline__ float ei_f32(double mu, float var, double best) {
  const float sig = sqrtf(var);
  const float imp = (float)(best - mu);
  if (!(sig > 0.f)) return fmaxf(imp, 0.f);
  return sig * tau_f32(imp / sig);
}

// H9 key: EI >= +0 canonicalised (kills -0 and NaN), then (bits << 32) | (2^32-1 - idx).
__device__ __forceinline__ unsigned long long make_key(float ei, uint64_t gidx) {
  if (isnan(ei)) return 0ull;
  const float e = ei > 0.f ? ei : 0.f;
  return ((unsigned long long)__float_as_uint(e) << 32) |
         (unsigned long long)(0xFFFFFFFFu - (uint32_t)gidx);
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long k) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long q = __shfl_xor_sync(0xffffffffu, k, o);
    k = q > k ? q : k;
  }
  return k;
}

// Per-candidate epilogue: optional raw outputs (H11) and the CTA argmax -> atomicMax (H9).
// Must be called by every thread of the block (uniform search per block).
__device__ __forceinline__ void finish_candidate(const ScoreLaunch &p, int s,
                                                 const SearchMeta &m, bool valid,
                                                 int64_t row0, int64_t row, double mu, float var,
                                                 float ei) {
  __shared__ unsigned long long wk[32];
  unsigned long long key = valid ? make_key(ei, (uint64_t)(p.m_base[s] + row)) : 0ull;
  if (valid) {
    if (p.out_mu) p.out_mu[row0 + row] = (float)(m.mean + m.std * mu);
    if (p.out_var) p.out_var[row0 + row] = (float)(m.std * m.std * (double)var);
    if (p.out_ei) p.out_ei[row0 + row] = (float)(m.std * (double)ei);
  }
  key = warp_max_u64(key);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wk[warp] = key;
  __syncthreads();
  if (warp == 0) {
    unsigned long long k2 = lane < (int)(blockDim.x >> 5) ? wk[lane] : 0ull;
    k2 = warp_max_u64(k2);
    if (lane == 0 && k2) atomicMax(p.keys + s, k2);
  }
}

}  // namespace gpbo
