// Scoring operand images (tcgen05): their geometry and the pack body shared by pack_tc_kernel
// (score_tc.cu) and the one-CTA fit kernel's tail (fit.cu), which packs the image while L^-1 is
// still hot (no separate launch).
#pragma once
#include <cuda_fp16.h>

#include "gpbo_internal.cuh"
#include "score_tc.cuh"
#include "tc_prims.cuh"

namespace gpbo {

// B rows appended to every resident L^-1 panel (score_tc.cu): row n16 = alpha hi, n16 + 1 =
// |alpha| hi (both in the hi image only), n16 + 2 = alpha lo 2^11 (lo image only), rest zero, so
// the fp16x3 variance MMA also accumulates V[n16] = K* alpha_hi, V[n16 + 1] = K* |alpha| and
// V[n16 + 2] = K*_hi alpha_lo 2^11 (the mean of north star (b) "mu = K* alpha" on the tensor
// cores instead of FMAs in the K* epilogue).
constexpr int kMeanRows = 16;

struct TcGeom {
  int n16, kb, npan, off_l, off_a, off_w, img;
};

__host__ __device__ inline int align1k(int v) { return (v + 1023) & ~1023; }

__host__ __device__ inline TcGeom tc_geom(int n, int d) {
  TcGeom g;
  g.n16 = (n + 15) & ~15;
  g.kb = (d + 2 + 15) / 16;
  g.npan = (g.n16 + 31) / 32;
  // each 32-wide L^-1 panel carries 16 extra B rows after its n16 - 32 p rows: the mean rows
  // (see pack_body) that make the variance MMA also accumulate mu~ and sum K* |alpha|
  int lrows = 0;
  for (int p = 0; p < g.npan; ++p) lrows += g.n16 + kMeanRows - 32 * p;
  g.off_l = align1k(g.kb * 2 * g.n16 * 32);
  g.off_a = align1k(g.off_l + lrows * 128);
  g.off_w = g.off_a + g.n16 * 8;
  g.img = align1k(g.off_w + GPBO_MAX_D * 4);
  return g;
}


// CTA-pair layout (score_tc.cu, kPair): every search has two images of `half` bytes, one per CTA
// of the pair, each holding half of every B operand's rows (the MMA's N split):
//   [0, off_l)      X chunks: chunk q (training points [64 q, 64 q + N_q), N_q = min(64, n16 - 64 q)),
//                   K block k: hi (32 rows x 32 B) then lo, SWIZZLE_32B K-major; CTA r holds
//                   rows [64 q + r N_q / 2, + N_q / 2)
//   [off_l, off_w)  L^-1 + mean-row slabs, one per 16-wide k step s (k in [16 s, 16 s + 16)):
//                   rows j in [16 s, n16 + 16) (N_s = n16 + 16 - 16 s), CTA r holds rows
//                   [16 s + r N_s / 2, + N_s / 2) as hi (N_s / 2 x 32 B) then lo, SWIZZLE_32B
//   [off_w, half)   per-dimension candidate scales (GPBO_MAX_D floats)
struct TcPairGeom {
  int n16, kb, nchunk, nks, off_l, off_w, half;
};

// byte offset of k-step slab s in the L part: 32 sum_{s' < s} (nv16 - 16 s')
__host__ __device__ inline int tc_pair_slab(int nv16, int s) {
  return 32 * (s * nv16 - 8 * s * (s - 1));
}

__host__ __device__ inline TcPairGeom tc_pair_geom(int n, int d) {
  TcPairGeom g;
  g.n16 = (n + 15) & ~15;
  g.kb = (d + 2 + 15) / 16;
  g.nchunk = (g.n16 + 63) / 64;
  g.nks = g.n16 / 16;
  g.off_l = align1k(g.nchunk * g.kb * 2048);
  g.off_w = align1k(g.off_l + tc_pair_slab(g.n16 + kMeanRows, g.nks));
  g.half = align1k(g.off_w + GPBO_MAX_D * 4);
  return g;
}

// One CTA per search.  Scales (powers of two, exact): x^ = g x/l 2^-e with g = sqrt5 (Matern)
// or 1/sqrt2 (RBF) and e chosen so max(|x^*|^2 over the unit box, |x^_j|^2) <= 2^13;
// K* 2^tK <= 2^13; L^-1 2^uL <= 2^14.  V = L^-1 K* then carries 2^(tK + uL).
// meta_s: the search's meta record (global; the tcgen05 constants are written back by the block
// with write_meta), m: its current value; threads t0 = 0.. of stride tstep share every loop (all
// threads of the block must call: block barriers inside); sc[5], il2[GPBO_MAX_D]: shared scratch.
__device__ __forceinline__ void pack_body(SearchMeta *meta_s, SearchMeta m, const double *Linv64,
                                          const double *Xs64, const double *alpha64,
                                          const float *ls32, unsigned char *img_all, int t0,
                                          int tstep, bool write_meta, double *sc, double *il2) {
  if (!m.tc_ok || (m.status != GPBO_OK && m.status != GPBO_WDEGENERATE)) return;
  const int n = m.n, d = m.d;
  const TcGeom g = tc_geom(n, d);
  const TcsGeom gs = tcs_geom(n, d);
  const bool stream = m.tc_stream != 0;
  unsigned char *img = img_all + m.img_off;
  const double *Li = Linv64 + m.mat_off;
  const double *X = Xs64 + m.x_off;
  const double gk = m.kernel == GPBO_RBF ? 0.70710678118654752440 : 2.2360679774997896964;
  const double lmax = m.linv_absmax;
  // the lengthscale loads in parallel (thread 0 alone made d dependent global round trips)
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const double l = (double)ls32[m.ls_off + c];
    il2[c] = 1.0 / (l * l);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double qbox = 0.0;
    for (int c = 0; c < d; ++c) qbox += il2[c];
    const double Qm = fmax(gk * gk * qbox, gk * gk * (double)m.pmax);
    const int e = (int)ceil(0.5 * log2(fmax(Qm, 1e-30) / 8192.0));
    const int tK = (int)floor(log2(8192.0 / (double)m.sf2));
    const int uL = (int)floor(log2(16384.0 / fmax(lmax, 1e-300)));
    sc[0] = ldexp(gk, -e);   // x^ = x/l * sc0
    sc[1] = (double)e;
    sc[2] = (double)tK;
    sc[3] = (double)uL;
    const double sf2 = m.sf2;
    const double log2e = 1.4426950408889634074;
    const double c0 = ldexp(sf2, tK);
    if (m.kernel == GPBO_RBF) {
      m.c0 = (float)log2(c0);
      m.c1 = (float)(-ldexp(1.0, 2 * e) * log2e);
      m.c2 = m.c3 = 0.f;
    } else {
      m.c0 = (float)c0;
      m.c1 = (float)(-ldexp(1.0, e) * log2e);
      m.c2 = (float)ldexp(c0, e);
      m.c3 = (float)(ldexp(c0, 2 * e) / 3.0);
    }
    m.hscale = (float)ldexp(1.0, 2 * e);
    m.vunscale2 = (float)ldexp(1.0, -2 * (tK + uL));
    // mean rows: alpha 2^uA with max |alpha| 2^uA <= 2^14 (clamped so 2^-(tK + uA) is a normal
    // float); V[n16] then carries 2^(tK + uA)
    int uA = (int)floor(log2(16384.0 / fmax((double)m.alpha_max, 1e-300)));
    uA = max(-100 - tK, min(100 - tK, uA));
    sc[4] = (double)uA;
    m.munscale = (float)ldexp(1.0, -(tK + uA));
    m.pmax_h = (float)(gk * gk * (double)m.pmax);
    if (write_meta) *meta_s = m;
  }
  __syncthreads();
  const double xs = sc[0];
  const int e = (int)sc[1], tK = (int)sc[2], uL = (int)sc[3];
  auto put = [&](unsigned char *base_hi, unsigned char *base_lo, uint32_t off, double v) {
    const __half hi = __double2half(v);
    const __half lo = __double2half(v - (double)__half2float(hi));
    *reinterpret_cast<__half *>(base_hi + off) = hi;
    *reinterpret_cast<__half *>(base_lo + off) = lo;
  };
  const int uA = (int)sc[4];
  // one B-operand row j of the variance MMA at k-step column kk: L^-1 rows (j < n16) or the mean
  // rows (j = n16 + t), written as the hi / lo fp16 pair at `off` of the two blocks
  auto put_l = [&](unsigned char *bhi, unsigned char *blo, uint32_t off, int j, int kk) {
    if (j < g.n16) {
      const double v = (kk <= j && j < n) ? ldexp(Li[(size_t)j * n + kk], uL) : 0.0;
      put(bhi, blo, off, v);
      return;
    }
    const int t = j - g.n16;
    const double a = kk < n ? ldexp(alpha64[m.a_off + kk], uA) : 0.0;
    const __half ah = __double2half(a);
    __half vh = __double2half(0.0), vl = __double2half(0.0);
    if (t == 0) vh = ah;
    else if (t == 1) vh = __double2half(fabs(a));
    else if (t == 2) vl = __double2half(ldexp(a - (double)__half2float(ah), 11));
    *reinterpret_cast<__half *>(bhi + off) = vh;
    *reinterpret_cast<__half *>(blo + off) = vl;
  };
  // augmented training operand value [-2 x^_j, 1, |x^_j|^2] at (j, k)
  auto xval = [&](int j, int k) -> double {
    if (j >= n) return 0.0;
    if (k < d) return -2.0 * xs * X[(size_t)k * n + j];
    if (k == d) return 1.0;
    if (k == d + 1) {
      double pj = 0.0;
      for (int c = 0; c < d; ++c) pj += (xs * X[(size_t)c * n + j]) * (xs * X[(size_t)c * n + j]);
      return pj;
    }
    return 0.0;
  };
  if (m.tc_pair) {
    const TcPairGeom pg = tc_pair_geom(n, d);
    const int nv16 = pg.n16 + kMeanRows;
    // flat loops over both halves (every thread of the grid busy; per-slab loops left most of
    // them idle and serialised 2 x nks short passes)
    const int xe = pg.nchunk * pg.kb * 32 * 16;          // X elements per half
    for (int idx = t0; idx < 2 * xe; idx += tstep) {
      const int r = idx >= xe, e = idx - r * xe;
      const int k = e & 15, rr = (e >> 4) & 31, cb = e >> 9;  // cb = q kb + kblk
      const int q = cb / pg.kb, kblk = cb - q * pg.kb;
      const int h = min(64, pg.n16 - 64 * q) / 2;
      const double v = rr < h ? xval(64 * q + r * h + rr, 16 * kblk + k) : 0.0;
      unsigned char *hi = img + r * pg.half + cb * 2048;
      put(hi, hi + 1024, tc::sw_offset(rr, k * 2, 32), v);
    }
    const int le = tc_pair_slab(nv16, pg.nks) / 4;      // L elements per half (16 per row)
    for (int idx = t0; idx < 2 * le; idx += tstep) {
      const int r = idx >= le, e = idx - r * le;
      int s = 0;
      while (s + 1 < pg.nks && tc_pair_slab(nv16, s + 1) / 4 <= e) ++s;
      const int h = (nv16 - 16 * s) / 2, o = e - tc_pair_slab(nv16, s) / 4;
      const int rr = o >> 4, kk = o & 15;
      unsigned char *hi = img + r * pg.half + pg.off_l + tc_pair_slab(nv16, s);
      put_l(hi, hi + h * 32, tc::sw_offset(rr, kk * 2, 32), 16 * s + r * h + rr, 16 * s + kk);
    }
    for (int c = t0; c < 2 * GPBO_MAX_D; c += tstep) {
      const int r = c >= GPBO_MAX_D, cc = c - r * GPBO_MAX_D;
      float *wp = reinterpret_cast<float *>(img + r * pg.half + pg.off_w);
      wp[cc] = cc < d ? (float)(xs / (double)ls32[m.ls_off + cc]) : 0.f;
    }
    return;
  }
  // augmented training operand [-2 x^_j, 1, |x^_j|^2], K blocks of 16, rows n16
  for (int idx = t0; idx < g.n16 * g.kb * 16; idx += tstep) {
    const int j = idx / (g.kb * 16), k = idx % (g.kb * 16);
    const double v = xval(j, k);
    const int kblk = k >> 4;
    if (stream) {  // chunk-major: chunk q, K block, hi / lo blocks of 64 rows x 32 B
      unsigned char *hi = img + (((j >> 6) * g.kb + kblk) * 2) * 2048;
      put(hi, hi + 2048, tc::sw_offset(j & 63, (k & 15) * 2, 32), v);
    } else {
      unsigned char *hi = img + kblk * 2 * g.n16 * 32;
      put(hi, hi + g.n16 * 32, tc::sw_offset(j, (k & 15) * 2, 32), v);
    }
  }
  if (stream) {
    // L^-1 slabs in the streamed kernel's consumption order (score_tc.cuh)
    int off = gs.off_l;
    for (int w = 0; w < gs.nw; ++w) {
      for (int pp = 0; pp < tcs_window_panels(gs.n16, w); ++pp) {
        const int R = tcs_slab_rows(gs.n16, w, pp);
        const int r0 = tcs_window_end(gs.n16, w) - R;
        unsigned char *hi = img + off;
        for (int idx = t0; idx < R * 32; idx += tstep) {
          const int r = idx >> 5, k = idx & 31;
          const int j = r0 + r, kk = 32 * pp + k;
          const double v = (kk <= j && j < n) ? ldexp(Li[(size_t)j * n + kk], uL) : 0.0;
          put(hi, hi + R * 64, tc::sw_offset(r, k * 2, 64), v);
        }
        off += R * 128;
      }
    }
    float2 *ap = reinterpret_cast<float2 *>(img + gs.off_a);
    for (int j = t0; j < gs.n16; j += tstep) {
      const double a = j < n ? alpha64[m.a_off + j] : 0.0;
      ap[j] = make_float2((float)ldexp(a, -tK), (float)ldexp(fabs(a), -tK));
    }
    float *wp = reinterpret_cast<float *>(img + gs.off_w);
    for (int c = t0; c < GPBO_MAX_D; c += tstep)
      wp[c] = c < d ? (float)(xs / (double)ls32[m.ls_off + c]) : 0.f;
    return;
  }
  // L^-1 panels: panel p holds rows j in [32p, n16), k in [32p, 32p + 32), then the kMeanRows
  // mean rows (j = n16 + t)
  for (int pp = 0; pp < g.npan; ++pp) {
    const int R = g.n16 + kMeanRows - 32 * pp;
    unsigned char *hi = img + g.off_l + (pp * (g.n16 + kMeanRows) - 16 * pp * (pp - 1)) * 128;
    for (int idx = t0; idx < R * 32; idx += tstep) {
      const int r = idx >> 5, k = idx & 31;
      put_l(hi, hi + R * 64, tc::sw_offset(r, k * 2, 64), 32 * pp + r, 32 * pp + k);
    }
  }
  float2 *ap = reinterpret_cast<float2 *>(img + g.off_a);
  for (int j = t0; j < g.n16; j += tstep) {
    const double a = j < n ? alpha64[m.a_off + j] : 0.0;
    ap[j] = make_float2((float)ldexp(a, -tK), (float)ldexp(fabs(a), -tK));
  }
  float *wp = reinterpret_cast<float *>(img + g.off_w);
  for (int c = t0; c < GPBO_MAX_D; c += tstep)
    wp[c] = c < d ? (float)(xs / (double)ls32[m.ls_off + c]) : 0.f;
  (void)e;
}


}  // namespace gpbo
