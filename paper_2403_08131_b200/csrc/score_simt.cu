// H6-H9 on CUDA cores (float32, mean accumulated in float64): the correctness-first scoring
// kernel.  One thread per candidate; the candidate's row of K* lives in shared memory
// (column-major tile, conflict-free), the variance contraction v = L^-1 k* streams the float32
// (L^-1)^T rows through L1 as warp-uniform (broadcast) float4 loads.
//
// Formulas (readings R3-R5, R10 of DESIGN.md):
//   mu~ = k*^T alpha,  s2~ = max(sf2 - |L^-1 k*|^2, 0),  EI = s~ tau((best - mu~)/s~)
//   key = (bits(EI) << 32) | (2^32 - 1 - global_idx), per-search atomicMax  (H9)
#include <cmath>

#include "gpbo_internal.cuh"
#include "score_common.cuh"

namespace gpbo {
namespace {

template <int DMAX, int TM>
__global__ void __launch_bounds__(TM)
score_simt_kernel(const ScoreLaunch p) {
  extern __shared__ float ks[];  // [n_pad][TM]
  const int t = blockIdx.x;
  int lo = 0, hi = p.S;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (p.tile_first[mid] <= t) lo = mid; else hi = mid;
  }
  const int s = lo;
  const SearchMeta &mref = p.meta[s];
  const int n = mref.n, d = mref.d, d_pad = mref.d_pad, n_pad = mref.n_pad;
  const float sf2 = mref.sf2;
  const int kind = mref.kernel;
  if (mref.status != GPBO_OK && mref.status != GPBO_WDEGENERATE) return;  // failed fit

  const int64_t row0 = p.m_off[s];
  const int64_t Ms = p.m_off[s + 1] - row0;
  const int64_t row = (int64_t)(t - p.tile_first[s]) * TM + threadIdx.x;
  const bool valid = row < Ms;

  const float *ls = p.ls32 + mref.ls_off;
  float xs[DMAX];
  const float *xr = p.Xstar + p.x_off[s] + (valid ? row : 0) * d;
#pragma unroll
  for (int c = 0; c < DMAX; ++c) xs[c] = (valid && c < d) ? __fdiv_rn(__ldg(xr + c), ls[c]) : 0.f;

  // ---- H6: K* row and the mean (float64 accumulation of float32 K* x float64 alpha)
  const float *Xs = p.Xs32 + mref.xs_off;
  const double *alpha = p.alpha64 + mref.a_off;
  double mu = 0.0;
  float a1 = 0.f;  // sum_j |K*_j alpha_j|: scale of the mean's rounding error
  for (int j = 0; j < n; ++j) {
    float r2 = 0.f;
#pragma unroll
    for (int c = 0; c < DMAX; ++c) {
      if (c < d_pad) {
        const float diff = xs[c] - __ldg(Xs + j * d_pad + c);
        r2 = fmaf(diff, diff, r2);
      }
    }
    const float k = kernel_f32(r2, sf2, kind);
    ks[j * TM + threadIdx.x] = k;
    const double aj = __ldg(alpha + j);
    mu = fma((double)k, aj, mu);
    a1 = fmaf(k, fabsf((float)aj), a1);
  }

  // ---- H7: s2 = |L^-1 k*|^2 in blocks of 8 columns of (L^-1)^T
  const float *LT = p.LT32 + mref.lt_off;
  float s2 = 0.f;
  for (int jb = 0; jb < n; jb += 8) {
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.f;
    const int kmax = min(jb + 8, n);
    for (int k = 0; k < kmax; ++k) {
      const float a = ks[k * TM + threadIdx.x];
      const float4 l0 = __ldg(reinterpret_cast<const float4 *>(LT + (size_t)k * n_pad + jb));
      const float4 l1 = __ldg(reinterpret_cast<const float4 *>(LT + (size_t)k * n_pad + jb + 4));
      acc[0] = fmaf(a, l0.x, acc[0]); acc[1] = fmaf(a, l0.y, acc[1]);
      acc[2] = fmaf(a, l0.z, acc[2]); acc[3] = fmaf(a, l0.w, acc[3]);
      acc[4] = fmaf(a, l1.x, acc[4]); acc[5] = fmaf(a, l1.y, acc[5]);
      acc[6] = fmaf(a, l1.z, acc[6]); acc[7] = fmaf(a, l1.w, acc[7]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) s2 = fmaf(acc[q], acc[q], s2);
  }

  // ---- H8 + H9 (fast phase): error bounds, then EI bracket / refine flagging.
  // K* relative error <= (5/6) dr2 + ~(s + 10) u with dr2 <= 2 (d + 3) u (|x*|^2 + |x_j|^2) for
  // the float32 direct differences; kappa factors are margins.
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < DMAX; ++c) q = fmaf(xs[c], xs[c], q);
  const float u = 5.9604645e-8f;
  float dmu = 0.2f * u * a1 * (2.f * (float)(d + 3) * (q + mref.pmax) + 64.f) * p.bound_scale;
  if (p.mean64 != nullptr && mref.mean_tier && valid) {  // precise-mean tier (mean64.cu)
    mu = p.mean64[row0 + row];
    dmu = 1e-12f * a1 * p.bound_scale;
  }
  const float var = fmaxf(sf2 - s2, 0.f);
  const float dvar = var_bound(u, sf2, s2, n, mref.linv_rowsum) * p.bound_scale;
  finish_fast(p, s, valid, row0, row, mu, dmu, var, dvar);
}

template <int DMAX, int TM>
cudaError_t launch_t(const ScoreLaunch &p, int tiles, int nmax, cudaStream_t st) {
  const int n_pad = (nmax + 63) & ~63;
  const int smem = n_pad * TM * (int)sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(score_simt_kernel<DMAX, TM>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  score_simt_kernel<DMAX, TM><<<tiles, TM, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_score_simt(const ScoreLaunch &p, int total_tiles, int dmax, int nmax,
                              cudaStream_t stream) {
  if (total_tiles <= 0) return cudaSuccess;
  if (dmax <= 8) return launch_t<8, kSimtTile>(p, total_tiles, nmax, stream);
  if (dmax <= 16) return launch_t<16, kSimtTile>(p, total_tiles, nmax, stream);
  if (dmax <= 32) return launch_t<32, kSimtTile>(p, total_tiles, nmax, stream);
  return launch_t<64, kSimtTile>(p, total_tiles, nmax, stream);
}

}  // namespace gpbo
