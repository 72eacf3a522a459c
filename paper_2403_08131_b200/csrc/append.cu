// O(n^2) append update of a fitted model for sequential BO.
//
// The BO loop of the paper re-trains the surrogate after every new evaluation (PAPER.md L72,
// §III.A: "re-training the surrogate model"; L249/L256: its O(N^3) cost).  With the
// hyper-parameters fixed, the new Gram matrix is the old one bordered by one row and column,
//     K' = [K  k; k^T  kappa],  k = k(X, x_new),  kappa = sf2 + sn2 + j   (same jitter j),
// whose Cholesky factor and inverse follow from the old ones in O(n^2) (bordered Cholesky):
//     l = L^-1 k,   delta = sqrt(kappa - |l|^2),   L' = [L 0; l^T delta],
//     L'^-1 = [L^-1 0; -(l^T L^-1) / delta  1/delta].
// This is exactly the factor a full refactorisation at the same jitter produces (the bordered
// matrix's leading block is K, and Cholesky is unique), up to float64 rounding.  The targets are
// re-standardised over the n + 1 values (reading R7), then w = L'^-1 y~, alpha = L'^-T w and the
// diagnostics are recomputed (O(n^2)).  delta^2 <= 0 (K' not positive definite at this jitter)
// asks the caller for a full refit with the jitter ladder (status ENOTPD, jitter_k = -2).
// One CTA per search; float64 throughout.
#include <cmath>

#include "gpbo_internal.cuh"

namespace gpbo {
namespace {

constexpr int kAppendThreads = 512;
constexpr int kAW = kAppendThreads / 32;

__device__ __forceinline__ double kval(double r2, double sf2, int kind) {
  if (kind == GPBO_RBF) return sf2 * exp(-0.5 * r2);
  const double r = sqrt(r2);
  const double s5 = 2.23606797749978969640917366873;
  return sf2 * (1.0 + s5 * r + (5.0 / 3.0) * r2) * exp(-s5 * r);
}

// Deterministic block reduction (fixed tree order); op 0 = sum, 1 = max, 2 = min.
__device__ double breduce(double v, double *red, int op) {
  auto f = [op](double a, double b) { return op == 0 ? a + b : op == 1 ? fmax(a, b) : fmin(a, b); };
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = f(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = red[0];
  for (int i = 1; i < kAW; ++i) t = f(t, red[i]);
  return t;
}

__global__ void __launch_bounds__(kAppendThreads)
append_kernel(const SearchMeta *__restrict__ meta_in, const AppendIO io,
              SearchMeta *__restrict__ meta_out) {
  __shared__ double xs[GPBO_MAX_D];     // x_new / l
  __shared__ double kv[GPBO_MAX_N];     // k(X, x_new), later y~
  __shared__ double lv[GPBO_MAX_N];     // l = L^-1 k, later w = L'^-1 y~
  __shared__ double red[kAW];
  __shared__ int bad_s;
  const int s = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const SearchMeta P = io.prev_meta[s];
  SearchMeta m = meta_in[s];
  const int n = P.n, n1 = n + 1, d = P.d;
  const double sf2 = P.sf2, sn2 = P.sn2;
  const float *xn = io.x_new + m.ls_off;  // x_new of search s: d values, offsets as ls
  const double ynew = io.y_new[s];
  // ---- inputs: validate and copy the old arrays into the new layout (appending x_new, y_new)
  if (tid == 0) bad_s = !isfinite(ynew);
  __syncthreads();
  for (int c = tid; c < d; c += kAppendThreads) {
    const float l = io.prev_ls32[P.ls_off + c];
    if (!isfinite(xn[c])) bad_s = 1;
    io.ls32[m.ls_off + c] = l;
    xs[c] = (double)xn[c] / (double)l;
  }
  __syncthreads();
  if (bad_s) {
    if (tid == 0) { m.status = GPBO_EINVAL; m.jitter_k = -1; m.lml = -INFINITY; meta_out[s] = m; }
    return;
  }
  for (int e = tid; e < n * d; e += kAppendThreads) io.X32[m.x_off + e] = io.prev_X32[P.x_off + e];
  for (int c = tid; c < d; c += kAppendThreads) io.X32[m.x_off + (int64_t)n * d + c] = xn[c];
  for (int i = tid; i < n; i += kAppendThreads) io.y64[m.y_off + i] = io.prev_y64[P.y_off + i];
  if (tid == 0) io.y64[m.y_off + n] = ynew;
  for (int e = tid; e < d * n1; e += kAppendThreads) {  // x / l, column-major d x n1
    const int c = e / n1, i = e - c * n1;
    io.Xs64[m.x_off + e] = i < n ? io.prev_Xs64[P.x_off + (int64_t)c * n + i] : xs[c];
  }
  // ---- k = k(X, x_new) by direct differences (reading R1), kappa = sf2 + sn2 + j
  const double *Xp = io.prev_Xs64 + P.x_off;
  for (int j = tid; j < n; j += kAppendThreads) {
    double r2 = 0.0;
    for (int c = 0; c < d; ++c) {
      const double t = xs[c] - Xp[(int64_t)c * n + j];
      r2 = fma(t, t, r2);
    }
    kv[j] = kval(r2, sf2, P.kernel);
  }
  double q = 0.0;
  for (int c = tid; c < d; c += kAppendThreads) q = fma(xs[c], xs[c], q);
  const double pnew = breduce(q, red, 0);  // |x_new / l|^2 (includes the barrier for kv)
  const double kappa = sf2 + sn2 + P.jitter;
  // ---- l = L^-1 k: warp per row (L^-1 row-major, lanes over the row)
  const double *Li = io.prev_Linv64 + P.mat_off;
  for (int i = warp; i < n; i += kAW) {
    double a = 0.0;
    for (int j = lane; j <= i; j += 32) a = fma(Li[(int64_t)i * n + j], kv[j], a);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) lv[i] = a;
  }
  __syncthreads();
  double ll = 0.0;
  for (int i = tid; i < n; i += kAppendThreads) ll = fma(lv[i], lv[i], ll);
  ll = breduce(ll, red, 0);
  const double d2 = kappa - ll;
  if (!(d2 > 0.0) || !isfinite(d2)) {  // not positive definite at this jitter: full refit
    if (tid == 0) { m.status = GPBO_ENOTPD; m.jitter_k = -2; m.lml = -INFINITY; meta_out[s] = m; }
    return;
  }
  const double delta = sqrt(d2), idelta = 1.0 / delta;
  // ---- L' (column-major, lower part) and L'^-1 (row-major, lower part)
  const double *Lp = io.prev_L64 + P.mat_off;
  double *Ln = io.L64 + m.mat_off, *Lin = io.Linv64 + m.mat_off;
  for (int64_t e = tid; e < (int64_t)n * n; e += kAppendThreads) {
    const int j = (int)(e / n), i = (int)(e - (int64_t)j * n);  // L: column j, row i
    if (i >= j) Ln[(int64_t)j * n1 + i] = Lp[e];
  }
  for (int64_t e = tid; e < (int64_t)n * n; e += kAppendThreads) {
    const int i = (int)(e / n), j = (int)(e - (int64_t)i * n);  // L^-1: row i, column j
    if (j <= i) Lin[(int64_t)i * n1 + j] = Li[e];
  }
  for (int j = tid; j < n; j += kAppendThreads) Ln[(int64_t)j * n1 + n] = lv[j];
  if (tid == 0) { Ln[(int64_t)n * n1 + n] = delta; Lin[(int64_t)n * n1 + n] = idelta; }
  // new row of L^-1: t_j = -(sum_{i >= j} l_i (L^-1)_ij) / delta, thread per column (coalesced
  // over j for each row i)
  double rabs = tid == 0 ? idelta : 0.0, rmax = idelta;
  for (int j = tid; j < n; j += kAppendThreads) {
    double a = 0.0;
    for (int i = j; i < n; ++i) a = fma(lv[i], Li[(int64_t)i * n + j], a);
    const double t = -a * idelta;
    Lin[(int64_t)n * n1 + j] = t;
    rabs += fabs(t);
    rmax = fmax(rmax, fabs(t));
  }
  rabs = breduce(rabs, red, 0);  // the new row's abs sum (1/delta counted once)
  rmax = breduce(rmax, red, 1);
  // ---- H1 over the n + 1 targets (ddof 0; reading R7 / R7a as the fit)
  const double *y = io.y64 + m.y_off;
  __syncthreads();  // y64 / L'^-1 writes visible to the block
  double acc = 0.0, amax = 0.0;
  for (int i = tid; i < n1; i += kAppendThreads) { acc += y[i]; amax = fmax(amax, fabs(y[i])); }
  const double mean = breduce(acc, red, 0) / n1;
  amax = breduce(amax, red, 1);
  acc = 0.0;
  for (int i = tid; i < n1; i += kAppendThreads) { const double t = y[i] - mean; acc += t * t; }
  double stdv = sqrt(breduce(acc, red, 0) / n1);
  const bool degenerate = !(stdv > 1e-12 * amax);
  if (degenerate) stdv = 1.0;
  double bmin = INFINITY;
  for (int i = tid; i < n1; i += kAppendThreads) {
    const double t = degenerate ? 0.0 : (y[i] - mean) / stdv;
    kv[i] = t;  // y~
    bmin = fmin(bmin, t);
  }
  const double best = breduce(bmin, red, 2);  // (barrier: y~ complete)
  // ---- w = L'^-1 y~ (warp per row), log det, |w|^2
  double ww = 0.0, ld = 0.0;
  for (int i = warp; i < n1; i += kAW) {
    double a = 0.0;
    for (int j = lane; j <= i; j += 32) a = fma(Lin[(int64_t)i * n1 + j], kv[j], a);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) {
      lv[i] = a;
      ww = fma(a, a, ww);
      ld -= log(Lin[(int64_t)i * n1 + i]);
    }
  }
  ww = breduce(ww, red, 0);
  ld = breduce(ld, red, 0);
  // ---- alpha = L'^-T w (thread per column), |alpha|_1, max |alpha|
  double l1 = 0.0, amx = 0.0;
  double *alpha = io.alpha64 + m.a_off;
  for (int j = tid; j < n1; j += kAppendThreads) {
    double a = 0.0;
    for (int i = j; i < n1; ++i) a = fma(Lin[(int64_t)i * n1 + j], lv[i], a);
    alpha[j] = a;
    l1 += fabs(a);
    amx = fmax(amx, fabs(a));
  }
  for (int j = n1 + tid; j < m.n_pad; j += kAppendThreads) alpha[j] = 0.0;
  l1 = breduce(l1, red, 0);
  amx = breduce(amx, red, 1);
  if (tid == 0) {
    m.sf2 = P.sf2; m.sn2 = P.sn2;
    m.status = degenerate ? GPBO_WDEGENERATE : GPBO_OK;
    m.jitter_k = P.jitter_k; m.jitter = P.jitter;
    m.mean = mean; m.std = stdv; m.best = best; m.alpha_l1 = l1;
    m.pmax = (float)fmax((double)P.pmax, pnew);
    m.alpha_max = (float)amx;
    m.linv_rowsum = fmaxf(P.linv_rowsum, (float)rabs);
    m.linv_absmax = fmax(P.linv_absmax, rmax);
    m.lml = -0.5 * ww - ld - 0.5 * n1 * 1.8378770664093454836;
    m.mean_tier = sf2 * l1 > kMeanTierL1 ? 1 : 0;
    meta_out[s] = m;
  }
}

}  // namespace

cudaError_t launch_append(const SearchMeta *meta_in, int S, const AppendIO &io,
                          SearchMeta *meta_out, cudaStream_t stream) {
  append_kernel<<<S, kAppendThreads, 0, stream>>>(meta_in, io, meta_out);
  return cudaGetLastError();
}

}  // namespace gpbo
