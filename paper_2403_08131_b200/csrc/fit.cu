// H1-H4 of the hot path: standardise y, Gram matrix, jittered Cholesky,
// triangular inverse, alpha -- one CTA per sub-search, float64 throughout.
//
// PAPER.md L249/L256 (§IV.D): the GP's "O(N^3) training complexity" is this factorisation.
// The kernel/jitter/standardisation readings are R1, R2, R7, R9 of DESIGN.md.
//
// Layout: the working matrix A is the lower triangle of an n x n float64 matrix, column-major
// (column j contiguous from its diagonal down).  For n <= kFitSmemMaxN it lives in shared memory,
// packed (column j starts at j n - j (j - 1) / 2, 216 KB at n = 232); otherwise the CTA works in
// place, unpacked, in the model's global Linv64 buffer (L2 resident).  Accesses go through the
// column-base function cb(j) and generic pointers, so the same code serves both cases.
#include <cmath>

#include "gpbo_internal.cuh"

namespace gpbo {
namespace {

constexpr int kWarps = kFitThreads / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reductions (fixed tree order).
template <class Op>
__device__ double block_reduce(double v, double *red, Op op, double identity) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < kWarps ? red[lane] : identity;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = op(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  double r = red[32];
  __syncthreads();
  return r;
}

struct AddOp { __device__ double operator()(double a, double b) const { return a + b; } };
struct MaxOp { __device__ double operator()(double a, double b) const { return fmax(a, b); } };
struct MinOp { __device__ double operator()(double a, double b) const { return fmin(a, b); } };

__device__ __forceinline__ double kernel_value(double r2, double sf2, int kind) {
  if (kind == GPBO_RBF) return sf2 * exp(-0.5 * r2);
  const double r = sqrt(r2);
  const double s5 = 2.23606797749978969640917366873;  // sqrt(5)
  return sf2 * (1.0 + s5 * r + (5.0 / 3.0) * r2) * exp(-s5 * r);
}

// The body is instantiated for a shared-memory (packed) and a global (unpacked) working matrix so
// that every access to A compiles to LDS/STS or LDG/STG instead of generic loads.
template <bool kSmem>
__device__ __forceinline__ void fit_body(double *sm, double *red,
                                         const SearchMeta *__restrict__ meta_in,
                                         const float *__restrict__ X32,
                                         const float *__restrict__ ls32,
                                         const double *__restrict__ y64, double *L64,
                                         double *Linv64, float *Xs32, double *Xs64, float *LT32,
                                         double *alpha64, SearchMeta *__restrict__ meta_out) {
  const int s = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  SearchMeta m = meta_in[s];
  const int n = m.n, d = m.d;
  const int nr = (n + 1) & ~1;
  double *yt = sm;
  double *tmp = sm + nr;
  double *w = sm + 2 * nr;
  double *A = kSmem ? sm + 3 * nr : Linv64 + m.mat_off;
  // A(i, j), i >= j, lives at A[cb(j) + i]
  auto cb = [&](int j) -> int { return kSmem ? j * n - (j * (j - 1)) / 2 - j : j * n; };
  const float *X = X32 + m.x_off;
  const float *ls = ls32 + m.ls_off;
  const double *y = y64 + m.y_off;

  // ---- input validation (GPBO_EINVAL on any non-finite / out-of-domain value)
  int bad = 0;
  for (int i = tid; i < n * d; i += kFitThreads) bad |= !isfinite(X[i]);
  for (int i = tid; i < n; i += kFitThreads) bad |= !isfinite(y[i]);
  for (int i = tid; i < d; i += kFitThreads) bad |= !(ls[i] > 0.f) || !isfinite(ls[i]);
  bad |= !(m.sf2 > 0.f) || !isfinite(m.sf2) || !(m.sn2 >= 0.f) || !isfinite(m.sn2);
  bad = __syncthreads_or(bad);
  if (bad) {
    if (tid == 0) { m.status = GPBO_EINVAL; m.jitter_k = -1; meta_out[s] = m; }
    return;
  }

  // ---- H1: y~ = (y - mean) / std, ddof = 0 (reading R7); degenerate -> y~ = 0, std = 1
  double acc = 0.0, amax = 0.0;
  for (int i = tid; i < n; i += kFitThreads) { acc += y[i]; amax = fmax(amax, fabs(y[i])); }
  const double mean = block_reduce(acc, red, AddOp(), 0.0) / n;
  amax = block_reduce(amax, red, MaxOp(), 0.0);
  acc = 0.0;
  for (int i = tid; i < n; i += kFitThreads) { const double t = y[i] - mean; acc += t * t; }
  double stdv = sqrt(block_reduce(acc, red, AddOp(), 0.0) / n);
  const bool degenerate = !(stdv > 1e-12 * amax);
  if (degenerate) stdv = 1.0;
  double bmin = INFINITY;
  for (int i = tid; i < n; i += kFitThreads) {
    const double t = degenerate ? 0.0 : (y[i] - mean) / stdv;
    yt[i] = t;
    bmin = fmin(bmin, t);
  }
  const double best = block_reduce(bmin, red, MinOp(), INFINITY);

  // ---- scoring operands: X / l in float32 (IEEE division), zero padded to n_pad x d_pad,
  // and in float64 (n x d) for the refine phase; pmax = max_j |x_j / l|^2
  for (int e = tid; e < m.n_pad * m.d_pad; e += kFitThreads) {
    const int i = e / m.d_pad, c = e - i * m.d_pad;
    Xs32[m.xs_off + e] = (i < n && c < d) ? __fdiv_rn(X[i * d + c], ls[c]) : 0.f;
  }
  double pm = 0.0;
  for (int i = tid; i < n; i += kFitThreads) {
    double q = 0.0;
    for (int c = 0; c < d; ++c) {
      const double v = (double)X[i * d + c] / (double)ls[c];
      Xs64[m.x_off + (size_t)c * n + i] = v;  // column-major: x/l of point i, dim c
      q += v * v;
    }
    pm = fmax(pm, q);
  }
  const double pmax = block_reduce(pm, red, MaxOp(), 0.0);

  // ---- H2 + H3: Gram matrix and Cholesky with the jitter ladder j_k = 1e-8 10^k sf2
  const double sf2 = m.sf2, sn2 = m.sn2;
  int jk = -1;
  double jit = 0.0;
  double p10 = 1.0;
  for (int k = 0; k < 7; ++k, p10 *= 10.0) {
    jit = 1e-8 * p10 * sf2;
    __syncthreads();
    for (int j = warp; j < n; j += kWarps) {
      const double *xc = Xs64 + m.x_off;  // column-major (d x n): coalesced across lanes
      for (int i = j + lane; i < n; i += 32) {
        // x / l precomputed in float64 above (the oracle's A / l, B / l then difference)
        double r2 = 0.0;
        for (int c = 0; c < d; ++c) {
          const double diff = xc[(size_t)c * n + i] - xc[(size_t)c * n + j];
          r2 += diff * diff;
        }
        double v = kernel_value(r2, sf2, m.kernel);
        if (i == j) v += sn2 + jit;
        A[cb(j) + i] = v;
      }
    }
    // right-looking column Cholesky, in place, lower triangle
    bool ok = true;
    for (int c = 0; c < n; ++c) {
      __syncthreads();
      double *Ac = A + cb(c);
      const double p = Ac[c];
      if (!(p > 0.0) || !isfinite(p)) { ok = false; break; }  // uniform across the CTA
      const double lcc = sqrt(p);
      const double rl = 1.0 / lcc;
      for (int i = c + 1 + tid; i < n; i += kFitThreads) Ac[i] *= rl;
      __syncthreads();
      if (tid == 0) Ac[c] = lcc;
      for (int j = c + 1 + warp; j < n; j += kWarps) {
        const double ljc = Ac[j];
        double *Aj = A + cb(j);
        for (int i = j + lane; i < n; i += 32) Aj[i] -= Ac[i] * ljc;
      }
    }
    if (ok) { jk = k; break; }
  }
  __syncthreads();
  if (jk < 0) {
    if (tid == 0) {
      m.status = GPBO_ENOTPD; m.jitter_k = -1; m.jitter = NAN;
      m.mean = mean; m.std = stdv; m.best = best; m.alpha_l1 = 0.0;
      meta_out[s] = m;
    }
    return;
  }
  // keep L (col-major, full) for diagnostics
  for (size_t e = tid; e < (size_t)n * n; e += kFitThreads) {
    const int j = (int)(e / n), i = (int)(e - (size_t)j * n);
    L64[m.mat_off + e] = (i >= j) ? A[cb(j) + i] : 0.0;
  }

  // ---- H4: in-place inverse X = L^-1 by a forward sweep over the rows of L (O(n) steps of
  // parallel rank-1 updates; critical path O(n)):  at step k, row k of X is final after
  // X[k][c] /= L[k][k]; then X[i][c] -= L[i][k] X[k][c] for i > k, c <= k (X[i][k] starts at 0).
  for (int k = 0; k < n; ++k) {
    __syncthreads();
    double *Ak = A + cb(k);
    const double lkk = Ak[k];
    for (int i = k + 1 + tid; i < n; i += kFitThreads) tmp[i] = Ak[i];  // column k of L
    __syncthreads();
    const double inv = 1.0 / lkk;
    // row k: X[k][c] = X[k][c] / L[k][k] for c < k (stored at (k, c)), X[k][k] = 1 / L[k][k]
    for (int c = tid; c <= k; c += kFitThreads) {
      double *p = A + cb(c) + k;
      *p = c == k ? inv : *p * inv;
    }
    __syncthreads();
    // rows i > k: X[i][c] = X[i][c] - L[i][k] X[k][c]  (c < k), X[i][k] = -L[i][k] X[k][k]
    for (int c = warp; c <= k; c += kWarps) {
      double *Ac = A + cb(c);
      const double xkc = Ac[k];
      if (c == k)
        for (int i = k + 1 + lane; i < n; i += 32) Ac[i] = -tmp[i] * xkc;
      else
        for (int i = k + 1 + lane; i < n; i += 32) Ac[i] -= tmp[i] * xkc;
    }
  }
  __syncthreads();
  // w = L^-1 y~
  for (int i = tid; i < n; i += kFitThreads) {
    double a2 = 0.0;
    for (int k = 0; k <= i; ++k) a2 += A[cb(k) + i] * yt[k];
    w[i] = a2;
  }
  __syncthreads();
  // alpha = L^-T w  (warp per k, lanes over i >= k)
  double l1 = 0.0, amx = 0.0;
  for (int k = warp; k < m.n_pad; k += kWarps) {
    double a2 = 0.0;
    if (k < n)
      for (int i = k + lane; i < n; i += 32) a2 += A[cb(k) + i] * w[i];
    a2 = warp_sum(a2);
    if (lane == 0) { alpha64[m.a_off + k] = a2; l1 += fabs(a2); amx = fmax(amx, fabs(a2)); }
  }
  l1 = block_reduce(l1, red, AddOp(), 0.0);
  amx = block_reduce(amx, red, MaxOp(), 0.0);
  double rs = 0.0, lam = 0.0;
  for (int j = tid; j < n; j += kFitThreads) {
    double a3 = 0.0;
    for (int k = 0; k <= j; ++k) {
      const double v = fabs(A[cb(k) + j]);
      a3 += v;
      lam = fmax(lam, v);
    }
    rs = fmax(rs, a3);
  }
  rs = block_reduce(rs, red, MaxOp(), 0.0);
  lam = block_reduce(lam, red, MaxOp(), 0.0);
  // write L^-1 (col-major) and the float32 (L^-1)^T scoring operand: LT[k][j] = Linv[j][k]
  if (kSmem)
    for (size_t e = tid; e < (size_t)n * n; e += kFitThreads) {
      const int j = (int)(e / n), i = (int)(e - (size_t)j * n);
      Linv64[m.mat_off + e] = (i >= j) ? A[cb(j) + i] : 0.0;
    }
  else
    for (size_t e = tid; e < (size_t)n * n; e += kFitThreads) {
      const int j = (int)(e / n), i = (int)(e - (size_t)j * n);
      if (i < j) A[e] = 0.0;
    }
  for (size_t e = tid; e < (size_t)m.n_pad * m.n_pad; e += kFitThreads) {
    const int k = (int)(e / m.n_pad), j = (int)(e - (size_t)k * m.n_pad);
    LT32[m.lt_off + e] = (k < n && j < n && j >= k) ? (float)A[cb(k) + j] : 0.f;
  }
  if (tid == 0) {
    m.status = degenerate ? GPBO_WDEGENERATE : GPBO_OK;
    m.jitter_k = jk; m.jitter = jit;
    m.mean = mean; m.std = stdv; m.best = best; m.alpha_l1 = l1;
    m.pmax = (float)pmax; m.alpha_max = (float)amx; m.linv_rowsum = (float)rs;
    m.linv_absmax = lam;
    meta_out[s] = m;
  }
}

__global__ void __launch_bounds__(kFitThreads, 1)
fit_kernel(const SearchMeta *__restrict__ meta_in, const float *__restrict__ X32,
           const float *__restrict__ ls32, const double *__restrict__ y64, double *L64,
           double *Linv64, float *Xs32, double *Xs64, float *LT32, double *alpha64,
           SearchMeta *__restrict__ meta_out) {
  extern __shared__ double sm[];
  __shared__ double red[33];
  if (meta_in[blockIdx.x].use_smem)
    fit_body<true>(sm, red, meta_in, X32, ls32, y64, L64, Linv64, Xs32, Xs64, LT32, alpha64,
                   meta_out);
  else
    fit_body<false>(sm, red, meta_in, X32, ls32, y64, L64, Linv64, Xs32, Xs64, LT32, alpha64,
                    meta_out);
}

}  // namespace

cudaError_t launch_fit(const SearchMeta *meta_d, int S, int smem_bytes, const float *X32,
                       const float *ls32, const double *y64, double *L64, double *Linv64,
                       float *Xs32, double *Xs64, float *LT32, double *alpha64,
                       SearchMeta *meta_out, cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(fit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_bytes);
  if (e != cudaSuccess) return e;
  fit_kernel<<<S, kFitThreads, smem_bytes, stream>>>(meta_d, X32, ls32, y64, L64, Linv64, Xs32,
                                                     Xs64, LT32, alpha64, meta_out);
  return cudaGetLastError();
}

}  // namespace gpbo
