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
#include <algorithm>
#include <atomic>
#include <cmath>

#include "gpbo_internal.cuh"
#include "score_tc_helpers.cuh"

namespace gpbo {
namespace {

// whether a search of the launch is in the precise tier (decided by the fit, possibly still
// pending on the host): the block's threads check the S records in parallel (a serial scan by
// every thread cost ~17 us per launch at S = 64 -- one dependent L2 round trip per search)
__device__ __forceinline__ bool any_mean_tier(const ScoreLaunch &p) {
  int any = 0;
  for (int i = threadIdx.x; i < p.S; i += blockDim.x) {
    const SearchMeta &m = p.meta[i];
    any |= m.mean_tier && (m.status == GPBO_OK || m.status == GPBO_WDEGENERATE);
  }
  return __syncthreads_or(any) != 0;
}

constexpr int kChunk = 64;
#ifndef GPBO_M64_RSQ32  // float32-seeded sqrt in kval64: measured slower (1.28 -> 1.35 ms), off
#define GPBO_M64_RSQ32 0
#endif
constexpr int kExpTab = 1024;  // e^{-k/16}, k < 1024 (arguments >= 64: e^-64 ~ 1.6e-28 -> 0)

// e^{-s} for s >= 0 in float64: s = k/16 + f, f in [0, 1/16): e^{-k/16} from the table times a
// degree-9 Taylor polynomial of e^{-f} (truncation (1/16)^10/10! ~ 2.6e-19)
__device__ __forceinline__ double exp_neg(double s, const double *tab) {
  const double t = s * 16.0;
  if (!(t < (double)kExpTab)) return 0.0;
  const int k = (int)t;
  const double f = -(s - (double)k * 0.0625);
  double p = 2.7557319223985893e-06;   // 1/9!
  p = fma(p, f, 2.4801587301587302e-05);  // 1/8!
  p = fma(p, f, 1.9841269841269841e-04);  // 1/7!
  p = fma(p, f, 1.3888888888888889e-03);  // 1/6!
  p = fma(p, f, 8.3333333333333333e-03);  // 1/5!
  p = fma(p, f, 4.1666666666666667e-02);  // 1/4!
  p = fma(p, f, 1.6666666666666667e-01);  // 1/3!
  p = fma(p, f, 0.5);
  p = fma(p, f, 1.0);
  p = fma(p, f, 1.0);
  return tab[k] * p;
}

// sqrt(r2) in float64 from the MUFU reciprocal square root refined by two Newton steps
__device__ __forceinline__ double sqrt_nr(double r2) {
  if (!(r2 > 0.0)) return r2 == 0.0 ? 0.0 : r2;  // 0 -> 0, NaN -> NaN
  double y;
#if GPBO_M64_RSQ32
  // float32 MUFU estimate (~2^-22; the float64 MUFU path is slower) when r2 is in float range
  if (r2 > 1e-30 && r2 < 1e30) {
    float yf;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"((float)r2));
    y = (double)yf;
  } else {
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  }
#else
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
#endif
#pragma unroll
  for (int i = 0; i < 2; ++i) y = fma(0.5 * y, fma(-r2, y * y, 1.0), y);
  const double r = r2 * y;
  return fma(0.5 * y, fma(-r, r, r2), r);  // one correction of r itself
}

__device__ __forceinline__ double kval64(double r2, double sf2, int kind, const double *tab) {
  if (kind == GPBO_RBF) return sf2 * exp_neg(0.5 * r2, tab);
  const double s = 2.23606797749978969640917366873 * sqrt_nr(r2);
  return sf2 * fma(s, fma(s, 1.0 / 3.0, 1.0), 1.0) * exp_neg(s, tab);
}

template <int DMAX>
__global__ void __launch_bounds__(128)
mean64_kernel(const ScoreLaunch p, const double *__restrict__ Xs64, const double *__restrict__ etab,
              int tile, int tile_lo, int tiles, double *mean64) {
  __shared__ __align__(16) double xs[kChunk][DMAX];
  __shared__ double qa[kChunk][2];  // |x_j / l|^2, alpha_j
  __shared__ double tab[kExpTab];
  // nothing to do unless a search of the launch is in the precise tier (decided by the fit,
  // possibly still pending on the host): one early exit per block of the persistent grid
  if (!any_mean_tier(p)) return;
  for (int e = threadIdx.x; e < kExpTab; e += blockDim.x) tab[e] = etab[e];
  for (int t = tile_lo + (int)blockIdx.x; t < tile_lo + tiles; t += gridDim.x) {
    const int s = search_of(p.tile_first, p.S, t);
    const SearchMeta &m = p.meta[s];
    if (!m.mean_tier || (m.status != GPBO_OK && m.status != GPBO_WDEGENERATE)) continue;
    const int n = m.n, d = m.d;
    const int64_t Ms = p.m_off[s + 1] - p.m_off[s];
    const int64_t row = (int64_t)(t - p.tile_first[s]) * tile + threadIdx.x;
    const bool valid = threadIdx.x < tile && row < Ms;
    const float *x = p.Xstar + p.x_off[s] + (valid ? row : 0) * d;
    const float *ls = p.ls32 + m.ls_off;
    double xr[DMAX];
    double q = 0.0;
#pragma unroll
    for (int c = 0; c < DMAX; ++c) {
      xr[c] = (valid && c < d) ? (double)x[c] / (double)ls[c] : 0.0;
      q = fma(xr[c], xr[c], q);  // NaN inputs stay NaN through q, dot and mu
    }
    const double *Xj = Xs64 + m.x_off;  // column-major d x n
    const double *alpha = p.alpha64 + m.a_off;
    const double sf2 = m.sf2;
    double mu = 0.0;
    for (int j0 = 0; j0 < n; j0 += kChunk) {
      const int cnt = min(kChunk, n - j0);
      __syncthreads();
      for (int e = threadIdx.x; e < kChunk * DMAX; e += blockDim.x) {
        const int j = e / DMAX, c = e - j * DMAX;
        xs[j][c] = (j < cnt && c < d) ? Xj[(int64_t)c * n + j0 + j] : 0.0;
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
        double d0 = 0.0, d1 = 0.0;  // two independent chains
        const double2 *xj = reinterpret_cast<const double2 *>(xs[j]);
#pragma unroll
        for (int c = 0; c < DMAX / 2; ++c) {
          const double2 v = xj[c];
          d0 = fma(xr[2 * c], v.x, d0);
          d1 = fma(xr[2 * c + 1], v.y, d1);
        }
        double r2 = q + qa[j][0] - 2.0 * (d0 + d1);
        r2 = r2 < 0.0 ? 0.0 : r2;  // (NaN propagates)
        mu = fma(kval64(r2, sf2, m.kernel, tab), qa[j][1], mu);
      }
    }
    if (valid) mean64[p.m_off[s] + row] = mu;
  }
}

// The same precise mean with the GEMM-form distances on the FP64 tensor cores (measured: config 2
// BO layout 1.50 -> 1.28 ms, config 4 BO 4.60 -> 3.22 ms; the kernel values on the FP64 pipe,
// latency-bound chains, are the rest): a CTA (8 warps)
// per scoring tile of <= 128 candidates, the training points in chunks of 64 staged in shared
// memory (x_j / l, |x_j / l|^2, alpha_j); warp w owns candidate blocks w and w + 8 (8 rows each):
// per 8-point block one DMMA m8n8k4 chain over the dimensions (the point block's B fragments
// shared by both candidate blocks) gives x* . x_j, then each lane evaluates the kernel for its
// (candidate, 2 points) and accumulates k alpha; lanes of a candidate reduce in a fixed order.
// The O(n d) distance work leaves the FP64 (DFMA) pipe for the tensor pipe; the kernel values
// stay on the FP64 pipe.
constexpr int kM64Warps = 8;

__device__ __forceinline__ void dmma64(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// row stride (doubles) >= d4 with stride = 4 (mod 8): a fragment load (rows gid < 4 of a
// half-warp, columns tig) hits distinct banks
__host__ __device__ __forceinline__ int m64_ld(int d4) { return (d4 % 8 == 4) ? d4 : d4 + 4; }

__global__ void __launch_bounds__(32 * kM64Warps)
mean64_dmma_kernel(const ScoreLaunch p, const double *__restrict__ Xs64,
                   const double *__restrict__ etab, int tile, int tile_lo, int tiles, int dmax,
                   double *mean64) {
  extern __shared__ __align__(16) double msm[];
  const int d4max = (dmax + 3) / 4 * 4, ld = m64_ld(d4max);
  double *tab = msm;                         // [kExpTab]
  double *xa = tab + kExpTab;                // [128][ld]   candidates x* / l
  double *xb = xa + 128 * ld;                // [kChunk][ld] training points x_j / l
  double *qb = xb + kChunk * ld;             // [kChunk]    |x_j / l|^2
  double *ab = qb + kChunk;                  // [kChunk]    alpha_j
  double *qa = ab + kChunk;                  // [128]       |x* / l|^2
  if (!any_mean_tier(p)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  for (int e = tid; e < kExpTab; e += 32 * kM64Warps) tab[e] = etab[e];
  for (int t = tile_lo + (int)blockIdx.x; t < tile_lo + tiles; t += gridDim.x) {
    const int s = search_of(p.tile_first, p.S, t);
    const SearchMeta &m = p.meta[s];
    if (!m.mean_tier || (m.status != GPBO_OK && m.status != GPBO_WDEGENERATE)) continue;
    const int n = m.n, d = m.d, d4 = (d + 3) / 4 * 4;
    const int64_t Ms = p.m_off[s + 1] - p.m_off[s];
    const int64_t row0 = (int64_t)(t - p.tile_first[s]) * tile;
    const int rows = (int)min((int64_t)tile, Ms - row0);
    const float *ls = p.ls32 + m.ls_off;
    const double *Xj = Xs64 + m.x_off;  // column-major d x n
    const double *alpha = p.alpha64 + m.a_off;
    const double sf2 = m.sf2;
    __syncthreads();  // the previous tile is done with xa / qa
    for (int e = tid; e < 128 * d4; e += 32 * kM64Warps) {
      const int r = e / d4, c = e - r * d4;
      xa[r * ld + c] = (r < rows && c < d)
          ? (double)p.Xstar[p.x_off[s] + (row0 + r) * d + c] / (double)ls[c] : 0.0;
    }
    __syncthreads();
    if (tid < 128) {
      double q = 0.0;
      for (int c = 0; c < d; ++c) q = fma(xa[tid * ld + c], xa[tid * ld + c], q);
      qa[tid] = q;  // (NaN inputs stay NaN through q, the distance and mu)
    }
    double mu[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // [candidate block][point of the lane's pair]
    for (int j0 = 0; j0 < n; j0 += kChunk) {
      const int cnt = min(kChunk, n - j0);
      __syncthreads();  // qa written; the previous chunk is consumed
      for (int e = tid; e < kChunk * d4; e += 32 * kM64Warps) {
        const int j = e / d4, c = e - j * d4;
        xb[j * ld + c] = (j < cnt && c < d) ? Xj[(int64_t)c * n + j0 + j] : 0.0;
      }
      for (int j = tid; j < kChunk; j += 32 * kM64Warps) {
        double qj = 0.0;
        if (j < cnt)
          for (int c = 0; c < d; ++c) {
            const double v = Xj[(int64_t)c * n + j0 + j];
            qj = fma(v, v, qj);
          }
        qb[j] = qj;
        ab[j] = j < cnt ? alpha[j0 + j] : 0.0;
      }
      __syncthreads();
      for (int J = 0; 8 * J < cnt; ++J) {
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        const double *bp = xb + (8 * J + gid) * ld + tig;
        for (int k0 = 0; k0 < d4; k0 += 4) {
          const double b = bp[k0];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int cb = warp + kM64Warps * h;
            dmma64(acc[h][0], acc[h][1], xa[(8 * cb + gid) * ld + k0 + tig], b);
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cb = warp + kM64Warps * h;
          const double q = qa[8 * cb + gid];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int j = 8 * J + 2 * tig + u;
            if (j < cnt) {
              double r2 = q + qb[j] - 2.0 * acc[h][u];
              r2 = r2 < 0.0 ? 0.0 : r2;  // (NaN propagates)
              mu[h][u] = fma(kval64(r2, sf2, m.kernel, tab), ab[j], mu[h][u]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double v = mu[h][0] + mu[h][1];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      const int r = 8 * (warp + kM64Warps * h) + gid;
      if (tig == 0 && r < rows) mean64[p.m_off[s] + row0 + r] = v;
    }
  }
}

}  // namespace

cudaError_t launch_mean64(const ScoreLaunch &p, const double *Xs64, int tile, int tile_lo,
                          int tiles, int dmax, double *mean64, const double *etab, int num_sms,
                          cudaStream_t stream) {
  if (tiles <= 0) return cudaSuccess;
#ifndef GPBO_MEAN64_DMMA
#define GPBO_MEAN64_DMMA 1
#endif
  if (GPBO_MEAN64_DMMA && tile <= 128) {
    const int d4max = (dmax + 3) / 4 * 4, ld = m64_ld(d4max);
    const size_t smem = ((size_t)kExpTab + 128 * ld + kChunk * ld + 2 * kChunk + 128) * sizeof(double);
    // the attribute is per device (one ctx per device may run in one process, on different
    // threads): a per-device flag, set once at the largest size
    static std::atomic<int> attr_done[64];
    int dev = 0;
    cudaError_t e0 = cudaGetDevice(&dev);
    if (e0 != cudaSuccess) return e0;
    if (smem > 48 * 1024 && (dev < 0 || dev >= 64 || !attr_done[dev].load())) {
      cudaError_t e = cudaFuncSetAttribute(mean64_dmma_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (e != cudaSuccess) return e;
      if (dev >= 0 && dev < 64) attr_done[dev].store(1);
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mean64_dmma_kernel, 32 * kM64Warps, smem);
    const int grid = std::min(tiles, num_sms * std::max(per_sm, 1));
    mean64_dmma_kernel<<<grid, 32 * kM64Warps, smem, stream>>>(p, Xs64, etab, tile, tile_lo, tiles,
                                                               dmax, mean64);
    return cudaGetLastError();
  }
  const int thr = tile <= 64 ? 64 : 128;
  const int grid = std::min(tiles, num_sms * 8);
#define GPBO_MEAN64(D)                                                                          \
  if (dmax <= D) {                                                                              \
    mean64_kernel<D><<<grid, thr, 0, stream>>>(p, Xs64, etab, tile, tile_lo, tiles, mean64);    \
    return cudaGetLastError();                                                                  \
  }
  GPBO_MEAN64(4) GPBO_MEAN64(8) GPBO_MEAN64(12) GPBO_MEAN64(16) GPBO_MEAN64(20) GPBO_MEAN64(24)
  GPBO_MEAN64(32) GPBO_MEAN64(40) GPBO_MEAN64(48) GPBO_MEAN64(56) GPBO_MEAN64(64)
#undef GPBO_MEAN64
  return cudaErrorInvalidValue;
}

// e^{-k/16}, k < kExpTab, in float64 (host std::exp; the device table of exp_neg)
void mean64_exp_table(double *host) {
  for (int k = 0; k < kExpTab; ++k) host[k] = std::exp(-k / 16.0);
}
int mean64_exp_table_size() { return kExpTab; }

}  // namespace gpbo
