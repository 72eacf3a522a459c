// Precise-mean tier of the fast phase (SURVEY.md §8(c) reading R13).
//
// The fast phase's float32 mean mu~ = K* alpha carries an error ~ u32 sum_j |K*_j alpha_j|.
// BO-like training sets (clustered near an incumbent) make alpha large with cancelling signs
// (|alpha|_1 ~ 1e3-1e5), so that error bound swamps the EI differences between candidates and
// the argmax filter flags nearly every candidate for the float64 refine (measured: 2^20 of 2^20 at
// config 2's BO layout, 213 ms per step).  The R13 reading's remedy is a mean tier chosen per
// fit: searches with sf2 |alpha|_1 > kMeanTierL1 get mu~ in float64 for every candidate from
// this kernel -- k(x*, x_j) by the GEMM-form distance |x*|^2 + |x_j|^2 - 2 x* . x_j in float64
// (cancellation ~1e-16 (|x*|^2 + |x_j|^2), far below what the argmax needs), the float64 kernel
// value and a float64 accumulation of k_j alpha_j -- and the fast phase uses it with a mean error
// bound of 1e-12 sum |k alpha|, so only the float32 variance's bound remains in the EI bracket.
// The O(n d) float64 work per candidate is the survey's "precise tier" (est. +100-200 % of the
// fast phase at n = 200-500); the O(n^2) variance contraction stays on the tensor cores.
//
// One thread per candidate row, a block per tile of the scoring launch's tiling (tile_first);
// the training points x_j / l (float64), |x_j / l|^2 and alpha_j are staged through shared
// memory in chunks of kChunk points (broadcast reads).  Searches of the fast tier exit at once.
#include <cmath>

#include "gpbo_internal.cuh"
#include "score_tc_helpers.cuh"

namespace gpbo {
namespace {

constexpr int kChunk = 64;

__device__ __forceinline__ double kval64(double r2, double sf2, int kind) {
  if (kind == GPBO_RBF) return sf2 * exp(-0.5 * r2);
  const double r = sqrt(r2);
  const double s5 = 2.23606797749978969640917366873;
  return sf2 * (1.0 + s5 * r + (5.0 / 3.0) * r2) * exp(-s5 * r);
}

template <int DMAX>
__global__ void __launch_bounds__(128)
mean64_kernel(const ScoreLaunch p, const double *__restrict__ Xs64, int tile, int tile_lo,
              double *mean64) {
  __shared__ double xs[kChunk][DMAX + 1];
  __shared__ double qa[kChunk][2];  // |x_j / l|^2, alpha_j
  const int t = tile_lo + (int)blockIdx.x;
  const int s = search_of(p.tile_first, p.S, t);
  const SearchMeta &m = p.meta[s];
  if (!m.mean_tier || (m.status != GPBO_OK && m.status != GPBO_WDEGENERATE)) return;
  const int n = m.n, d = m.d;
  const int64_t Ms = p.m_off[s + 1] - p.m_off[s];
  const int64_t row = (int64_t)(t - p.tile_first[s]) * tile + threadIdx.x;
  const bool valid = threadIdx.x < tile && row < Ms;
  const float *x = p.Xstar + p.x_off[s] + row * d;
  const float *ls = p.ls32 + m.ls_off;
  double xr[DMAX];
  double q = 0.0;
#pragma unroll
  for (int c = 0; c < DMAX; ++c) {
    xr[c] = (valid && c < d) ? (double)x[c] / (double)ls[c] : 0.0;
    q = fma(xr[c], xr[c], q);
  }
  const double *Xj = Xs64 + m.x_off;  // column-major d x n
  const double *alpha = p.alpha64 + m.a_off;
  const double sf2 = m.sf2;
  // padded coordinates c >= d stay 0 (they multiply zeros of xr; never NaN garbage)
  for (int e = threadIdx.x; e < kChunk * (DMAX + 1); e += blockDim.x) (&xs[0][0])[e] = 0.0;
  double mu = 0.0;
  for (int j0 = 0; j0 < n; j0 += kChunk) {
    const int cnt = min(kChunk, n - j0);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * d; e += blockDim.x) {
      const int c = e / cnt, j = e - c * cnt;
      xs[j][c] = Xj[(int64_t)c * n + j0 + j];
    }
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
      double qj = 0.0;
      for (int c = 0; c < d; ++c) {
        const double v = Xj[(int64_t)c * n + j0 + j];
        qj = fma(v, v, qj);
      }
      qa[j][0] = qj;
      qa[j][1] = alpha[j0 + j];
    }
    __syncthreads();
    for (int j = 0; j < cnt; ++j) {
      double dot = 0.0;
#pragma unroll
      for (int c = 0; c < DMAX; ++c) dot = fma(xr[c], xs[j][c], dot);  // padded c: xr = 0
      const double r2 = fmax(q + qa[j][0] - 2.0 * dot, 0.0);
      mu = fma(kval64(r2, sf2, m.kernel), qa[j][1], mu);
    }
  }
  if (valid) mean64[p.m_off[s] + row] = mu;
}

}  // namespace

cudaError_t launch_mean64(const ScoreLaunch &p, const double *Xs64, int tile, int tile_lo,
                          int tiles, int dmax, double *mean64, cudaStream_t stream) {
  if (tiles <= 0) return cudaSuccess;
  const int thr = tile <= 64 ? 64 : 128;
  // xs[j][c] needs d <= DMAX; padded coordinates multiply zeros
  if (dmax <= 8) mean64_kernel<8><<<tiles, thr, 0, stream>>>(p, Xs64, tile, tile_lo, mean64);
  else if (dmax <= 16) mean64_kernel<16><<<tiles, thr, 0, stream>>>(p, Xs64, tile, tile_lo, mean64);
  else if (dmax <= 32) mean64_kernel<32><<<tiles, thr, 0, stream>>>(p, Xs64, tile, tile_lo, mean64);
  else mean64_kernel<64><<<tiles, thr, 0, stream>>>(p, Xs64, tile, tile_lo, mean64);
  return cudaGetLastError();
}

}  // namespace gpbo
