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

// Error bound of the fast-phase variance sf2 - |v|^2 (v = L^-1 k* from float32 K*):
// empirically ~ u sqrt(n) (sf2 + |v|^2) (2 + 0.01 |L^-1|_inf sqrt(sf2)) on the bracket-test
// workloads; the factor 16 is the safety margin ("fast/refine split").
__device__ __forceinline__ float var_bound(float u, float sf2, float s2, int n, float linv_rs) {
  return 16.f * u * sqrtf((float)n) * (sf2 + s2) * (1.f + 0.01f * linv_rs * sqrtf(sf2));
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

// The incumbent in standardised units: the caller's raw-unit value (standardised with the fit's
// mean / std, which live on the device for an asynchronous fit), or NaN = the fitted best.
__device__ __forceinline__ double resolve_best(double best_in, const SearchMeta &m) {
  return isnan(best_in) ? m.best : (best_in - m.mean) / m.std;
}

// Epilogue of the fast phase for one candidate (every thread of the block calls it; the block
// belongs to one search).  mu: standardised fast mean (float32 K*), dmu: its error bound,
// var: standardised latent variance, dvar: its error bound.
//   kModeArgmax:    EI is bracketed by monotonicity of EI in (mu, sigma):
//                   EI_hi = EI(mu - dmu, var + dvar), EI_lo = EI(mu + dmu, var - dvar)
//                   (+-2e-4 relative for the float32 tau()).  The block max of EI_lo raises the
//                   search's running threshold; candidates with EI_hi >= threshold go to the
//                   refine list; candidates with EI_hi == 0 have EI == 0 exactly and settle
//                   their key here.
//   kModePosterior: store var~ for the dense refine pass.
//   kModeDebug:     store the phase's own values.
// The group of `nthreads` threads (warps gw0.. of the block, one candidate each) synchronises
// with named barrier `bar_id` (0 = the whole block).  force_refine: the fast phase could not
// evaluate this candidate safely (e.g. float16 range) -> EI_hi = +inf.
// Per-search values of the epilogue, loaded once per search segment by the persistent kernel
// (each is a dependent global round trip; the tcgen05 drain warps hoist them out of the tile
// loop).  thr: the search's running threshold as read by the caller for this tile.
struct FinishSeg {
  double best;      // incumbent, standardised
  int64_t m_base;   // global index of the search's first local candidate
  bool fitted;      // the (possibly asynchronous) fit succeeded
};

__device__ __forceinline__ FinishSeg finish_seg(const ScoreLaunch &p, int s) {
  const SearchMeta &mm = p.meta[s];
  FinishSeg f;
  f.fitted = mm.status == GPBO_OK || mm.status == GPBO_WDEGENERATE;
  f.best = resolve_best(p.best[s], mm);
  f.m_base = p.m_base[s];
  return f;
}

__device__ __forceinline__ float read_thr(const ScoreLaunch &p, int s) {
  return __uint_as_float(*(volatile const unsigned int *)(p.thr + s));
}

__device__ __forceinline__ void finish_fast(const ScoreLaunch &p, int s, const FinishSeg &fs,
                                            float thr, bool valid, int64_t row0, int64_t row,
                                            double mu, float dmu, float var, float dvar,
                                            bool force_refine, uint32_t bar_id, uint32_t nthreads,
                                            int gw0) {
  const bool fitted = fs.fitted;
  valid = valid && fitted;  // a failed asynchronous fit scores nothing
  const bool ok = valid && (force_refine || (isfinite(mu) && isfinite(var)));
  const double best = fs.best;
  float ei_lo = 0.f, ei_hi = 0.f;
  if (ok && p.mode != kModePosterior) {
    if (force_refine) {
      ei_hi = INFINITY;
      ei_lo = 0.f;
    } else {
      // Cheap screens (argmax mode), against the running threshold thr (a lower bound of the
      // search's final max EI_lo).  With s_hi = sqrt(var + dvar), z = (best - mu_lo)/s_hi:
      //   z < 0:  Gordon's inequality Phi(-x) >= x phi(x)/(1 + x^2) gives
      //           EI <= s_hi phi(z)/(1 + z^2)                       (one exp);
      //   z >= 0: Phi <= 1 gives EI <= s_hi phi(z) + (best - mu_lo)  (one exp).
      // A candidate whose screen is below thr cannot be the argmax: EI_hi := screen, EI_lo := 0
      // (both still valid bounds).  Otherwise EI_hi is evaluated exactly; EI_lo is needed only
      // when EI_hi >= thr (else it could neither raise the threshold nor be flagged).
      bool screened = false;
      if (p.mode == kModeArgmax) {
        // approximate sqrt / division / exp (relative errors ~1e-6, far inside the 1.001 margin):
        // this screen runs for every candidate on the drain warps, which share their
        // sub-partitions with the K* warps
        float s_hi;
        asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(s_hi) : "f"(var + dvar));
        const float imp = (float)(best - (mu - (double)dmu));
        const float z = __fdividef(imp, s_hi);
        if (s_hi > 0.f) {
          const float ph = s_hi * 0.398942280401432678f * __expf(-0.5f * z * z);
          const float ub = (z < 0.f ? __fdividef(ph, fmaf(z, z, 1.f)) : ph + imp) * 1.001f;
          if (ub < thr) { ei_hi = ub; ei_lo = 0.f; screened = true; }
        }
      }
      if (!screened) {
        ei_hi = ei_f32(mu - (double)dmu, var + dvar, best) * (1.f + 2e-4f);
        ei_lo = (p.mode != kModeArgmax || !(ei_hi < thr))
                    ? ei_f32(mu + (double)dmu, fmaxf(var - dvar, 0.f), best) * (1.f - 2e-4f)
                    : 0.f;
      }
    }
  }
  if (p.break_bracket) {  // test hook (gpbo_debug_bound_scale < 0): a deliberately wrong bracket
    ei_lo *= 0.5f;
    ei_hi *= 0.5f;
  }
  if (p.mode == kModePosterior) {
    if (valid) p.out_var[row0 + row] = var;
    return;
  }
  if (p.mode == kModeDebug) {
    if (valid) {
      const int64_t i = row0 + row;
      p.dbg_mu[i] = (float)mu; p.dbg_dmu[i] = dmu; p.dbg_var[i] = var; p.dbg_dvar[i] = dvar;
      p.dbg_eilo[i] = ok ? ei_lo : NAN; p.dbg_eihi[i] = ok ? ei_hi : NAN;
    }
    return;
  }
  __shared__ unsigned int s_thr[32];
  __shared__ unsigned long long s_zk[32];
  const unsigned int thr_entry = __float_as_uint(thr);
  const uint64_t gidx = (uint64_t)(fs.m_base + row);
  unsigned int lo_bits = ok ? __float_as_uint(fmaxf(ei_lo, 0.f)) : 0u;
  unsigned long long zkey = (ok && !(ei_hi > 0.f)) ? make_key(0.f, gidx) : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo_bits = max(lo_bits, __shfl_xor_sync(0xffffffffu, lo_bits, o));
    const unsigned long long q = __shfl_xor_sync(0xffffffffu, zkey, o);
    zkey = q > zkey ? q : zkey;
  }
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) - gw0, nw = nthreads >> 5;
  if (lane == 0) { s_thr[warp] = lo_bits; s_zk[warp] = zkey; }
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads) : "memory");
  if (warp == 0) {
    unsigned int lb = lane < nw ? s_thr[lane] : 0u;
    unsigned long long zk = lane < nw ? s_zk[lane] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lb = max(lb, __shfl_xor_sync(0xffffffffu, lb, o));
      const unsigned long long q = __shfl_xor_sync(0xffffffffu, zk, o);
      zk = q > zk ? q : zk;
    }
    if (lane == 0) {
      // fire-and-forget threshold update; the decision uses the global value read at entry
      // (any stale value <= the final threshold only flags more candidates)
      atomicMax(p.thr + s, lb);
      if (zk) atomicMax(p.keys + s, zk);
      s_thr[0] = max(thr_entry, lb);
    }
  }
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads) : "memory");
  const float thr_fin = __uint_as_float(s_thr[0]);
  const bool flag = ok && ei_hi > 0.f && ei_hi >= thr_fin;
  // audit sample of the candidates the filter excludes (their ei_hi bound is checked too)
  const bool audit = ok && !flag && ((uint32_t)gidx * 0x9E3779B1u) >> kAuditShift == 0u;
  const unsigned int mask = __ballot_sync(0xffffffffu, flag || audit);
  if (mask) {
    const int leader = __ffs(mask) - 1;
    unsigned int base = 0;
    if (lane == leader) base = atomicAdd(p.list_count, (unsigned int)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (flag || audit) {
      const unsigned int pos = base + __popc(mask & ((1u << lane) - 1u));
      if (pos < p.list_cap)
        p.list[pos] = RefineEntry{(uint32_t)s | (audit ? kEntryAudit : 0u), (uint32_t)row,
                                  ei_lo, ei_hi};
    }
  }
}

// Convenience form for kernels without a per-segment hoist (CUDA-core kernel): loads the
// search's values and the threshold itself.
__device__ __forceinline__ void finish_fast(const ScoreLaunch &p, int s, bool valid,
                                            int64_t row0, int64_t row, double mu, float dmu,
                                            float var, float dvar, bool force_refine = false,
                                            uint32_t bar_id = 0, uint32_t nthreads = 0,
                                            int gw0 = 0) {
  if (nthreads == 0) nthreads = blockDim.x;
  const FinishSeg fs = finish_seg(p, s);
  const float thr = p.mode == kModeArgmax ? read_thr(p, s) : 0.f;
  finish_fast(p, s, fs, thr, valid, row0, row, mu, dmu, var, dvar, force_refine, bar_id, nthreads,
              gw0);
}

}  // namespace gpbo
