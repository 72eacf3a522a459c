// Float64 refine phase of the scoring path (H6-H9 for the candidates that can still win).
//
// The fast phase (tcgen05 or CUDA-core kernel) evaluates K* in float32.  Its mean
// mu~ = k*^T alpha then carries an error ~ u32 sum_j |K*_j alpha_j|, which for ill-conditioned
// fits (|alpha|_1 >~ 1e3, reading R13) or for searches whose EI lives in the
// far tail is larger than the 1e-4 parity bar.  The fast phase therefore brackets every
// candidate's EI in [EI_lo, EI_hi]; only candidates with EI_hi >= max EI_lo (the running
// per-search threshold) are re-scored here, with the distance, the kernel value and the mean in
// float64 (the oracle's arithmetic: direct differences of x / l), the variance
// s2~ = sf2 - |L^-1 k*|^2 in float64 (in the far EI tail the float32 variance of the fast phase
// is not accurate enough: dEI/EI ~ z^2 ds2/(2 s2)), and EI's tau() in float64.
// The argmax key of a search is built only from refined EI values, so it is exact up to float64
// rounding and independent of how the candidates were sharded.
//
// gp_posterior runs the same code densely over all rows (posterior mode).
// One warp per candidate; lanes stride over the training points.
#include <algorithm>
#include <cmath>

#include "gpbo_internal.cuh"
#include "score_common.cuh"

namespace gpbo {
namespace {

constexpr int kRefineWarps = 8;

__device__ __forceinline__ double kernel64(double r2, double sf2, int kind) {
  if (kind == GPBO_RBF) return sf2 * exp(-0.5 * r2);
  const double r = sqrt(r2);
  const double s5 = 2.23606797749978969640917366873;
  return sf2 * (1.0 + s5 * r + (5.0 / 3.0) * r2) * exp(-s5 * r);
}

// tau(z) = phi(z) + z Phi(z) in float64 (erfcx form for z < 0, as in score_common.cuh).
__device__ __forceinline__ double tau64(double z) {
  const double inv_sqrt2pi = 0.398942280401432677939946059934;
  const double inv_sqrt2 = 0.707106781186547524400844362105;
  if (z >= 0.0) return inv_sqrt2pi * exp(-0.5 * z * z) + z * 0.5 * erfc(-z * inv_sqrt2);
  const double x = -z;
  return exp(-0.5 * z * z) * (inv_sqrt2pi - 0.5 * x * erfcx(x * inv_sqrt2));
}

__global__ void __launch_bounds__(kRefineWarps * 32)
refine_kernel(const RefineLaunch p) {
  __shared__ double xsh[kRefineWarps][GPBO_MAX_D];
  __shared__ double ksh[kRefineWarps][GPBO_MAX_N];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nent = p.list ? (int64_t)*p.list_count : p.dense_rows;
  for (int64_t e = (int64_t)blockIdx.x * kRefineWarps + warp; e < nent;
       e += (int64_t)gridDim.x * kRefineWarps) {
    int s;
    uint32_t row;
    float var;
    if (p.list) {
      const RefineEntry en = p.list[e];
      if (en.ei_hi < __uint_as_float(p.thr[en.s])) continue;  // cannot be the argmax
      s = en.s; row = en.row; var = en.var;
    } else {
      s = p.dense_s; row = (uint32_t)e; var = p.dense_var[e];
    }
    const SearchMeta &m = p.meta[s];
    const int n = m.n, d = m.d;
    const float *x = p.Xstar + p.x_off[s] + (int64_t)row * d;
    const float *ls = p.ls32 + m.ls_off;
    for (int c = lane; c < d; c += 32) xsh[warp][c] = (double)x[c] / (double)ls[c];
    __syncwarp();
    const double *Xj = p.Xs64 + m.x_off;
    const double *alpha = p.alpha64 + m.a_off;
    double mu = 0.0;
    for (int j = lane; j < n; j += 32) {
      double r2 = 0.0;
      for (int c = 0; c < d; ++c) {
        const double diff = xsh[warp][c] - Xj[j * d + c];
        r2 += diff * diff;
      }
      const double k = kernel64(r2, (double)m.sf2, m.kernel);
      ksh[warp][j] = k;
      mu += k * alpha[j];
    }
    __syncwarp();
    // v = L^-1 k*: lane owns rows j; Linv64 is column-major (column k contiguous over j)
    const double *Li = p.Linv64 + m.mat_off;
    double vv = 0.0;
    for (int j = lane; j < n; j += 32) {
      double v = 0.0;
      for (int k = 0; k <= j; ++k) v = fma(Li[(size_t)k * n + j], ksh[warp][k], v);
      vv = fma(v, v, vv);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mu += __shfl_xor_sync(0xffffffffu, mu, o);
      vv += __shfl_xor_sync(0xffffffffu, vv, o);
    }
    (void)var;
    if (lane == 0) {
      const double var64 = fmax((double)m.sf2 - vv, 0.0);
      const double sig = sqrt(var64);
      const double imp = p.best[s] - mu;
      const double ei = sig > 0.0 ? sig * tau64(imp / sig) : fmax(imp, 0.0);
      if (p.list) {
        const unsigned long long key = make_key((float)ei, (uint64_t)(p.m_base[s] + row));
        if (key) atomicMax(p.keys + s, key);
      } else {
        if (p.out_mu) p.out_mu[e] = (float)(m.mean + m.std * mu);
        if (p.out_var) p.out_var[e] = (float)(m.std * m.std * var64);
        if (p.out_ei) p.out_ei[e] = (float)(m.std * ei);
      }
    }
    __syncwarp();
  }
}

}  // namespace

cudaError_t launch_refine(const RefineLaunch &p, int64_t max_entries, int num_sms,
                          cudaStream_t stream) {
  if (max_entries <= 0) return cudaSuccess;
  const int64_t want = (max_entries + kRefineWarps - 1) / kRefineWarps;
  const int grid = (int)std::min<int64_t>(want, (int64_t)num_sms * 8);
  refine_kernel<<<grid, kRefineWarps * 32, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace gpbo
