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
// One CTA per candidate; threads stride over training points, then over rows of L^-1.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "gpbo_internal.cuh"
#include "score_common.cuh"

namespace gpbo {
namespace {

constexpr int kRefineThreads = 256;

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

// The fast phase's EI bracket must contain the float64 EI (up to float32 rounding of the
// bounds); anything else means an error bound failed and the argmax filter may have dropped the
// winner -- the caller re-scores the search exactly (api.cu, argmax_tail).
__device__ __forceinline__ bool bracket_violated(double ei, float lo, float hi) {
  return ei > (double)hi * (1.0 + 1e-6) + 1e-37 || ei < (double)lo * (1.0 - 1e-6) - 1e-37;
}

__device__ __forceinline__ double block_sum2(double v, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < kRefineThreads / 32; ++i) t += red[i];
  return t;
}

// One CTA per candidate: lanes over training points for K*, rows of L^-1 for v = L^-1 k*.
__global__ void __launch_bounds__(kRefineThreads)
refine_kernel(const RefineLaunch p) {
  __shared__ double xsh[GPBO_MAX_D];
  __shared__ double ksh[GPBO_MAX_N];
  __shared__ double red[kRefineThreads / 32];
  const int tid = threadIdx.x;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the fast phase's outputs are complete
  const int64_t nent = p.list ? (int64_t)*p.list_count : p.dense_rows;
  for (int64_t e = blockIdx.x; e < nent; e += gridDim.x) {
    int s;
    uint32_t row;
    RefineEntry en{};
    if (p.list) {
      en = p.list[e];
      s = (int)(en.s & ~kEntryAudit);
      // cannot be the argmax (uniform over the block); audit entries are always checked
      if (!(en.s & kEntryAudit) && en.ei_hi < __uint_as_float(p.thr[s])) continue;
      row = en.row;
    } else {
      s = p.dense_s; row = (uint32_t)e;
    }
    const SearchMeta &m = p.meta[s];
    const int n = m.n, d = m.d;
    const float *x = p.Xstar + p.x_off[s] + (int64_t)row * d;
    const float *ls = p.ls32 + m.ls_off;
    __syncthreads();  // previous candidate done with xsh / ksh
    for (int c = tid; c < d; c += kRefineThreads) xsh[c] = (double)x[c] / (double)ls[c];
    __syncthreads();
    const double *Xj = p.Xs64 + m.x_off;
    const double *alpha = p.alpha64 + m.a_off;
    double mu = 0.0;
    for (int j = tid; j < n; j += kRefineThreads) {
      double r2 = 0.0, r2b = 0.0;
      int c = 0;
      for (; c + 2 <= d; c += 2) {  // two independent loads per step
        const double d0 = xsh[c] - Xj[(size_t)c * n + j];  // column-major x/l
        const double d1 = xsh[c + 1] - Xj[(size_t)(c + 1) * n + j];
        r2 += d0 * d0;
        r2b += d1 * d1;
      }
      if (c < d) {
        const double d0 = xsh[c] - Xj[(size_t)c * n + j];
        r2 += d0 * d0;
      }
      r2 += r2b;
      const double k = kernel64(r2, (double)m.sf2, m.kernel);
      ksh[j] = k;
      mu += k * alpha[j];
    }
    mu = block_sum2(mu, red);  // includes the barrier that publishes ksh
    // v = L^-1 k*: warp per row j (Linv64 is row-major: lanes read consecutive k); four rows per
    // pass and the k loop unrolled by two, so up to 8 loads per lane are in flight (the rows come
    // from L2 / HBM: a pass is one memory round trip)
    const double *Li = p.Linv64 + m.mat_off;
    const int lane = tid & 31, wp = tid >> 5;
    constexpr int kW = kRefineThreads / 32;
    double vv = 0.0;
    for (int j0 = wp; j0 < n; j0 += 4 * kW) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      const double *row[4];
      int jr[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        jr[r] = j0 + r * kW < n ? j0 + r * kW : -1;  // -1: no such row
        row[r] = Li + (size_t)min(j0 + r * kW, n - 1) * n;
      }
      const int jmax = min(j0 + 3 * kW, n - 1);
      for (int k = lane; k <= jmax; k += 32) {  // the 4 rows' loads issue together
        const double kv = ksh[k];
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (k <= jr[r]) acc[r] = fma(row[r][k], kv, acc[r]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (j0 + r * kW < n) vv = fma(acc[r], acc[r], vv);
    }
    if (lane != 0) vv = 0.0;
    vv = block_sum2(vv, red);
    if (tid == 0) {
      // a non-finite candidate row (NaN / inf input, or a row masked by the generator's dedup)
      // makes mu or |v|^2 non-finite: it is never a suggestion and its outputs are NaN (fmax
      // would otherwise turn NaN into sig = 0, EI = 0 and a valid key)
      const bool fin = isfinite(mu) && isfinite(vv);
      const double var64 = fmax((double)m.sf2 - vv, 0.0);
      const double sig = sqrt(var64);
      const double imp = resolve_best(p.best[s], m) - mu;
      const double ei = !fin ? NAN : sig > 0.0 ? sig * tau64(imp / sig) : fmax(imp, 0.0);
      if (p.list || p.dense_keys) {
        const unsigned long long key = fin ? make_key((float)ei, (uint64_t)(p.m_base[s] + row)) : 0ull;
        if (key) atomicMax(p.keys + s, key);
        if (p.list && fin && bracket_violated(ei, en.ei_lo, en.ei_hi)) atomicAdd(p.viol + s, 1ull);
      } else {
        if (p.out_mu) p.out_mu[e] = fin ? (float)(m.mean + m.std * mu) : NAN;
        if (p.out_var) p.out_var[e] = fin ? (float)(m.std * m.std * var64) : NAN;
        if (p.out_ei) p.out_ei[e] = fin ? (float)(m.std * ei) : NAN;
      }
    }
  }
}

// Argmax-mode refine with a thread-block cluster of kSplit CTAs per flagged candidate: every CTA
// forms k* (and mu~) for all training points, then the rows of v = L^-1 k* are dealt to the
// CTAs (row j to CTA j mod kSplit) so the L^-1 stream (n^2 / 2 float64 from L2: 160 KB at
// n = 200, 1 MB at n = 500) is read by kSplit SMs at once; the partial |v|^2 go to CTA 0's shared
// memory (DSMEM) and are summed there in rank order (deterministic), and CTA 0 forms EI and the
// key.  The fast phase's final threshold is fixed while this runs, so every CTA of a cluster
// takes the same skip decision.
// kSplit = 4 for n <= 256, 8 above (measured: config 2 refine 0.023 -> 0.020 ms with 4, config
// 4 0.037 -> 0.046 with 4; 2 slower for both)
template <int kSplit>
__global__ void __cluster_dims__(kSplit, 1, 1) __launch_bounds__(kRefineThreads)
refine_split_kernel(const RefineLaunch p) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double xsh[GPBO_MAX_D];
  __shared__ double ksh[GPBO_MAX_N];
  __shared__ double red[kRefineThreads / 32];
  __shared__ double part[kSplit];
  const int tid = threadIdx.x;
  const int rank = (int)cluster.block_rank();
  const int64_t cid = blockIdx.x / kSplit, ncl = gridDim.x / kSplit;
  double *part0 = cluster.map_shared_rank(part, 0);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the fast phase's list is complete
  const int64_t nent = (int64_t)*p.list_count;
  for (int64_t e = cid; e < nent; e += ncl) {
    const RefineEntry en = p.list[e];
    const int s = (int)(en.s & ~kEntryAudit);
    // uniform over the cluster; audit entries are always checked
    if (!(en.s & kEntryAudit) && en.ei_hi < __uint_as_float(p.thr[s])) continue;
    const uint32_t row = en.row;
    const SearchMeta &m = p.meta[s];
    const int n = m.n, d = m.d;
    const float *x = p.Xstar + p.x_off[s] + (int64_t)row * d;
    const float *ls = p.ls32 + m.ls_off;
    __syncthreads();
    for (int c = tid; c < d; c += kRefineThreads) xsh[c] = (double)x[c] / (double)ls[c];
    __syncthreads();
    const double *Xj = p.Xs64 + m.x_off;
    const double *alpha = p.alpha64 + m.a_off;
    double mu = 0.0;
    for (int j = tid; j < n; j += kRefineThreads) {
      double r2 = 0.0, r2b = 0.0;
      int c = 0;
      for (; c + 2 <= d; c += 2) {
        const double d0 = xsh[c] - Xj[(size_t)c * n + j];
        const double d1 = xsh[c + 1] - Xj[(size_t)(c + 1) * n + j];
        r2 += d0 * d0;
        r2b += d1 * d1;
      }
      if (c < d) {
        const double d0 = xsh[c] - Xj[(size_t)c * n + j];
        r2 += d0 * d0;
      }
      r2 += r2b;
      const double k = kernel64(r2, (double)m.sf2, m.kernel);
      ksh[j] = k;
      mu += k * alpha[j];
    }
    mu = block_sum2(mu, red);
    // this CTA's rows j = rank + kSplit (w + kW i): warp per row, four rows per pass
    const double *Li = p.Linv64 + m.mat_off;
    const int lane = tid & 31, wp = tid >> 5;
    constexpr int kW = kRefineThreads / 32;
    double vv = 0.0;
    for (int jb = wp; rank + kSplit * jb < n; jb += 4 * kW) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      const double *rowp[4];
      int jr[4];
      int jmax = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int j = rank + kSplit * (jb + r * kW);
        jr[r] = j < n ? j : -1;
        rowp[r] = Li + (size_t)min(j, n - 1) * n;
        if (j < n) jmax = max(jmax, j);
      }
      for (int k = lane; k <= jmax; k += 32) {
        const double kv = ksh[k];
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (k <= jr[r]) acc[r] = fma(rowp[r][k], kv, acc[r]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (jr[r] >= 0) vv = fma(acc[r], acc[r], vv);
    }
    if (lane != 0) vv = 0.0;
    vv = block_sum2(vv, red);
    if (tid == 0) part0[rank] = vv;
    cluster.sync();  // the partials have landed in CTA 0
    if (rank == 0 && tid == 0) {
      double v2 = 0.0;
      for (int r = 0; r < kSplit; ++r) v2 += part[r];
      const bool fin = isfinite(mu) && isfinite(v2);  // non-finite rows: no key (refine_kernel)
      const double var64 = fmax((double)m.sf2 - v2, 0.0);
      const double sig = sqrt(var64);
      const double imp = resolve_best(p.best[s], m) - mu;
      const double ei = sig > 0.0 ? sig * tau64(imp / sig) : fmax(imp, 0.0);
      const unsigned long long key = fin ? make_key((float)ei, (uint64_t)(p.m_base[s] + row)) : 0ull;
      if (key) atomicMax(p.keys + s, key);
      if (fin && bracket_violated(ei, en.ei_lo, en.ei_hi)) atomicAdd(p.viol + s, 1ull);
    }
    cluster.sync();  // CTA 0 has read the partials before the next entry overwrites them
  }
}

// Argmax-mode refine for n <= 128 (config 3: ~5,000 entries of 64 searches): a WARP per entry
// instead of a CTA -- lane l owns training points / rows l + 32 q (q < 4): k*_j by direct
// differences (x* / l broadcast by shuffles), the float64 kernel and alpha_j k*_j, then
// v_j = sum_{i <= j} (L^-1)_ji k*_i with k*_i broadcast by shuffles (each lane walks its own rows
// of the row-major L^-1), warp sums for mu~ and |v|^2, lane 0 forms EI, the key and the bracket
// check -- no block barriers, 8 entries in flight per CTA.
constexpr int kRwWarps = 8;

__global__ void __launch_bounds__(32 * kRwWarps)
refine_warp_kernel(const RefineLaunch p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the fast phase's list is complete
  const int lane = threadIdx.x & 31;
  const int64_t nent = (int64_t)*p.list_count;
  const int64_t wstep = (int64_t)gridDim.x * kRwWarps;
  for (int64_t e = (int64_t)blockIdx.x * kRwWarps + (threadIdx.x >> 5); e < nent; e += wstep) {
    const RefineEntry en = p.list[e];
    const int s = (int)(en.s & ~kEntryAudit);
    if (!(en.s & kEntryAudit) && en.ei_hi < __uint_as_float(p.thr[s])) continue;  // (warp-uniform)
    const SearchMeta &m = p.meta[s];
    const int n = m.n, d = m.d;
    const float *x = p.Xstar + p.x_off[s] + (int64_t)en.row * d;
    const float *ls = p.ls32 + m.ls_off;
    const double *Xj = p.Xs64 + m.x_off;  // column-major x / l
    const double *alpha = p.alpha64 + m.a_off;
    const double xa = lane < d ? (double)x[lane] / (double)ls[lane] : 0.0;
    const double xb = lane + 32 < d ? (double)x[lane + 32] / (double)ls[lane + 32] : 0.0;
    double r2[4] = {0.0, 0.0, 0.0, 0.0};
    for (int c = 0; c < d; ++c) {
      const double xc = __shfl_sync(0xffffffffu, c < 32 ? xa : xb, c & 31);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = lane + 32 * q;
        if (j < n) { const double t = xc - Xj[(size_t)c * n + j]; r2[q] = fma(t, t, r2[q]); }
      }
    }
    const double sf2 = (double)m.sf2;
    double k[4], mu = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = lane + 32 * q;
      k[q] = j < n ? kernel64(r2[q], sf2, m.kernel) : 0.0;
      if (j < n) mu = fma(k[q], alpha[j], mu);
    }
    const double *Li = p.Linv64 + m.mat_off;  // row-major, lower part
    double v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int qb = 0; qb < 4; ++qb) {
      if (32 * qb >= n) break;
      // unrolled by 8 with predicates (not a break): the next columns' loads are in flight
      // while the FMAs of this one wait (a single entry's latency bounds small refine lists)
#pragma unroll 8
      for (int ii = 0; ii < 32; ++ii) {
        const int i = 32 * qb + ii;
        const double ki = __shfl_sync(0xffffffffu, k[qb], ii);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = lane + 32 * q;
          if (i < n && i <= j && j < n) v[q] = fma(Li[(size_t)j * n + i], ki, v[q]);
        }
      }
    }
    double vv = v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mu += __shfl_xor_sync(0xffffffffu, mu, o);
      vv += __shfl_xor_sync(0xffffffffu, vv, o);
    }
    if (lane == 0) {
      const bool fin = isfinite(mu) && isfinite(vv);  // non-finite rows: no key (refine_kernel)
      const double var64 = fmax(sf2 - vv, 0.0);
      const double sig = sqrt(var64);
      const double imp = resolve_best(p.best[s], m) - mu;
      const double ei = sig > 0.0 ? sig * tau64(imp / sig) : fmax(imp, 0.0);
      const unsigned long long key = fin ? make_key((float)ei, (uint64_t)(p.m_base[s] + en.row)) : 0ull;
      if (key) atomicMax(p.keys + s, key);
      if (fin && bracket_violated(ei, en.ei_lo, en.ei_hi)) atomicAdd(p.viol + s, 1ull);
    }
  }
}

// Small problems (rows x n16^2 small, n <= 64): the whole scoring in float64 -- no operand image,
// no fast phase, no refine list; exact up to float64 rounding (the oracle's arithmetic).  One
// warp per candidate: lane j owns training points j and j + 32 (k*_j by direct differences of
// x / l, the kernel, alpha_j k*_j) and rows j, j + 32 of v = L^-1 k* (k*_i broadcast by shuffle);
// warp sums give mu~ and |v|^2, lane 0 forms EI.  Keys (argmax mode; one atomic per block and
// search) or dense raw mu / var / EI (posterior mode).
constexpr int kDirectWarps = 8;

__global__ void __launch_bounds__(32 * kDirectWarps)
direct_kernel(const RefineLaunch p, int S, int64_t rows) {
  __shared__ unsigned long long skey[kDirectWarps];
  __shared__ int ss[kDirectWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t g = (int64_t)blockIdx.x * kDirectWarps + wid;  // candidate (warp-uniform)
  const bool posterior = p.out_mu || p.out_var || p.out_ei;
  unsigned long long key = 0ull;
  int s = 0;
  if (g < rows) {
    int lo = 0, hi = S;  // search of row g: m_off[s] <= g < m_off[s + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (p.m_off[mid] <= g) lo = mid; else hi = mid;
    }
    s = lo;
    while (s + 1 < S && p.m_off[s + 1] <= g) ++s;  // empty searches
    const SearchMeta &m = p.meta[s];
    if (m.status == GPBO_OK || m.status == GPBO_WDEGENERATE) {
      const int n = m.n, d = m.d;
      const int64_t row = g - p.m_off[s];
      const float *x = p.Xstar + p.x_off[s] + row * d;
      const float *ls = p.ls32 + m.ls_off;
      const double *Xj = p.Xs64 + m.x_off;  // column-major x / l
      const double *alpha = p.alpha64 + m.a_off;
      // x*_c / l_c for c = lane, lane + 32
      const double xa = lane < d ? (double)x[lane] / (double)ls[lane] : 0.0;
      const double xb = lane + 32 < d ? (double)x[lane + 32] / (double)ls[lane + 32] : 0.0;
      const int j0 = lane, j1 = lane + 32;
      double r0 = 0.0, r1 = 0.0;
      for (int c = 0; c < d; ++c) {
        const double xc = __shfl_sync(0xffffffffu, c < 32 ? xa : xb, c & 31);
        if (j0 < n) { const double t = xc - Xj[(size_t)c * n + j0]; r0 = fma(t, t, r0); }
        if (j1 < n) { const double t = xc - Xj[(size_t)c * n + j1]; r1 = fma(t, t, r1); }
      }
      const double sf2 = (double)m.sf2;
      const double k0 = j0 < n ? kernel64(r0, sf2, m.kernel) : 0.0;
      const double k1 = j1 < n ? kernel64(r1, sf2, m.kernel) : 0.0;
      double mu = (j0 < n ? k0 * alpha[j0] : 0.0) + (j1 < n ? k1 * alpha[j1] : 0.0);
      const double *Li = p.Linv64 + m.mat_off;  // row-major, lower part
      double v0 = 0.0, v1 = 0.0;
      for (int i = 0; i < n; ++i) {
        const double ki = __shfl_sync(0xffffffffu, i < 32 ? k0 : k1, i & 31);
        if (i <= j0 && j0 < n) v0 = fma(Li[(size_t)j0 * n + i], ki, v0);
        if (i <= j1 && j1 < n) v1 = fma(Li[(size_t)j1 * n + i], ki, v1);
      }
      double vv = v0 * v0 + v1 * v1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mu += __shfl_xor_sync(0xffffffffu, mu, o);
        vv += __shfl_xor_sync(0xffffffffu, vv, o);
      }
      if (lane == 0) {
        // non-finite rows (NaN input, dedup-masked candidates) are invalid: no key, NaN outputs
        // -- as the fast-phase kernels (kFlagInvalid / isfinite in finish_fast)
        const bool fin = isfinite(mu) && isfinite(vv);
        const double var64 = fmax(sf2 - vv, 0.0);
        const double sig = sqrt(var64);
        const double imp = resolve_best(p.best[s], m) - mu;
        const double ei = sig > 0.0 ? sig * tau64(imp / sig) : fmax(imp, 0.0);
        if (posterior) {
          if (p.out_mu) p.out_mu[g] = fin ? (float)(m.mean + m.std * mu) : NAN;
          if (p.out_var) p.out_var[g] = fin ? (float)(m.std * m.std * var64) : NAN;
          if (p.out_ei) p.out_ei[g] = fin ? (float)(m.std * ei) : NAN;
        } else if (fin) {
          key = make_key((float)ei, (uint64_t)(p.m_base[s] + row));
        }
      }
    }
  }
  if (posterior) return;
  if (lane == 0) { skey[wid] = key; ss[wid] = s; }
  __syncthreads();
  if (threadIdx.x == 0) {  // consecutive candidates: mostly one search per block
    unsigned long long acc = 0ull;
    const int s0 = ss[0];
    for (int w = 0; w < kDirectWarps; ++w) {
      if (ss[w] == s0) acc = skey[w] > acc ? skey[w] : acc;
      else if (skey[w]) atomicMax(p.keys + ss[w], skey[w]);
    }
    if (acc) atomicMax(p.keys + s0, acc);
  }
}

// gp_posterior's dense path: every row of search dense_s in float64 (the refine's arithmetic up
// to summation order: the float64 kernel, mu~ = k*^T alpha, s2~ = sf2 - |L^-1 k*|^2, tau), on the
// FP64 tensor cores, kPostTile = 32 candidates per CTA iteration:
//   1. x* / l of the tile and q* = |x* / l|^2 into shared memory;
//   2. K* from GEMM-form squared distances r^2 = q* + q - 2 (x* / l) . (x / l) on DMMA m8n8k4
//      (float64: the form's cancellation error ~ u q is ~1e-15 sf2 in k*, far inside T1, whose
//      variance term is relative to sf2 -- tests/helpers.py check_T1), clamped at 0 (NaN kept:
//      a non-finite candidate row yields NaN outputs); the kernel
//      in float64 on the fragments; K*^T into shared memory and the mean partials k* alpha;
//   3. V^T = L^-1 K*^T on DMMA: 8-row blocks J of L^-1 (2J + 2 k-steps of 4 each) dealt to the
//      warps by longest-processing-time (deterministic, near-equal k-step totals); A fragments
//      straight from L2 (row-major L^-1, lower part; four k-steps of loads in flight), B
//      fragments from the K*^T tile, four 8-candidate accumulators; |v|^2 accumulates per
//      candidate as each row block completes (V is never stored);
//   4. fixed-order reductions (deterministic), EI, raw outputs.
// Per candidate ~2 n d + n (n + 8) tensor flops plus the n kernel evaluations -- the
// per-candidate refine streams n^2 / 2 float64 of L^-1 per candidate instead.
constexpr int kPostTile = 32;
#ifndef GPBO_POST_PF
#define GPBO_POST_PF 8      // distance-stage B fragments in flight (k-steps of 4 dims)
#endif
#ifndef GPBO_POST_MINB
#define GPBO_POST_MINB 3    // resident CTAs per SM the 8-warp variant is compiled for
#endif
#ifndef GPBO_POST_PF8
#define GPBO_POST_PF8 4     // the same for the 8-warp variant
#endif
#ifndef GPBO_POST_ACC8
#define GPBO_POST_ACC8 1    // V accumulator sets (k-step parity) of the 8-warp variant (16 warps: 2)
#endif
#ifndef GPBO_POST_WSMALL
#define GPBO_POST_WSMALL 8  // warps per CTA for n <= 256
#endif
constexpr int kPostLd = kPostTile + 4;  // K*^T row stride (doubles): conflict-free B fragments

__device__ __forceinline__ void dmma64(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// kPostWarps: 8 (up to 3 CTAs per SM) or 16 when the K*^T tile limits the SM to one CTA (n > 256)
template <int kPostWarps>
__global__ void __launch_bounds__(32 * kPostWarps, kPostWarps == 8 ? GPBO_POST_MINB : 1)
posterior64_kernel(const RefineLaunch p, int dmax) {
  constexpr int kPostThreads = 32 * kPostWarps;
  constexpr int kGroups = kPostWarps / 4;  // point-block groups of the distance stage
  constexpr int kPF = kPostWarps == 8 ? GPBO_POST_PF8 : GPBO_POST_PF;
  constexpr int kAcc = kPostWarps == 8 ? GPBO_POST_ACC8 : 2;
  extern __shared__ __align__(16) double psm[];
  const int s = p.dense_s;
  const SearchMeta &m = p.meta[s];
  const int n = m.n, d = m.d, nt = (n + 7) / 8, n8 = 8 * nt, d4 = (d + 3) / 4 * 4;
  const int xld = (dmax + 3) / 4 * 4 + 1;
  double *ks = psm;                                  // [n8][kPostLd]: K*^T(j, c)
  double *xs = ks + (size_t)n8 * kPostLd;            // [kPostTile][xld]: x* / l (0 beyond d)
  double *qj = xs + (size_t)kPostTile * xld;         // [n8]: |x_j / l|^2
  double *qc = qj + n8;                              // [kPostTile]: |x* / l|^2
  double *red = qc + kPostTile;                      // [2][kPostWarps][kPostTile]
  int *owner = reinterpret_cast<int *>(red + 2 * kPostWarps * kPostTile);  // [nt]: warp of J
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const double *Xj = p.Xs64 + m.x_off;      // column-major d x n
  const double *alpha = p.alpha64 + m.a_off;
  const double *Li = p.Linv64 + m.mat_off;  // row-major, lower part
  const float *ls = p.ls32 + m.ls_off;
  const double sf2 = (double)m.sf2;
  const double best = resolve_best(p.best[s], m);
  // per-CTA setup: q_j, and the row-block -> warp deal (longest first to the least loaded)
  for (int j = tid; j < n8; j += kPostThreads) {
    double q = 0.0;
    if (j < n)
      for (int dim = 0; dim < d; ++dim) { const double v = Xj[(size_t)dim * n + j]; q = fma(v, v, q); }
    qj[j] = q;
  }
  if (tid == 0) {
    int load[kPostWarps];
    for (int q = 0; q < kPostWarps; ++q) load[q] = 0;
    for (int J = nt - 1; J >= 0; --J) {
      int w = 0;
      for (int q = 1; q < kPostWarps; ++q) w = load[q] < load[w] ? q : w;
      owner[J] = w;
      load[w] += 2 * J + 2;
    }
  }
  const int64_t ntile = (p.dense_rows + kPostTile - 1) / kPostTile;
  for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x) {
    const int64_t row0 = t * kPostTile;
    const int cnt = (int)min((int64_t)kPostTile, p.dense_rows - row0);
    __syncthreads();  // the previous tile is done with ks / xs / red (and the setup is visible)
    for (int e = tid; e < kPostTile * d4; e += kPostThreads) {
      const int cc = e / d4, dim = e - cc * d4;
      xs[cc * xld + dim] = cc < cnt && dim < d
          ? (double)p.Xstar[p.x_off[s] + (row0 + cc) * d + dim] / (double)ls[dim] : 0.0;
    }
    __syncthreads();
    if (tid < kPostTile) {
      double q = 0.0;
      for (int dim = 0; dim < d; ++dim) q = fma(xs[tid * xld + dim], xs[tid * xld + dim], q);
      qc[tid] = q;
    }
    __syncthreads();
    // 2. K* on DMMA: warp w -> candidate block cb = w & 3, point blocks J = (w >> 2) mod kGroups
    {
      const int cb = warp & 3;
      const double *xa = xs + (8 * cb + gid) * xld + tig;
      const double qa = qc[8 * cb + gid];
      double mu = 0.0;  // candidate 8 cb + gid, points 2 tig + {0, 1} of this warp's blocks
      for (int J = warp >> 2; J < nt; J += kGroups) {
        const int jb = 8 * J + gid;  // B column (point) of this lane's fragment loads
        const double *xb = Xj + min(jb, n - 1);
        // GPBO_POST_PF k-steps' B fragments in flight at once, then their DMMAs
        double d0 = 0.0, d1 = 0.0;
        for (int kb = 0; kb < d4; kb += 4 * kPF) {
          double bv[kPF];
#pragma unroll
          for (int u = 0; u < kPF; ++u) {
            const int dim = kb + 4 * u + tig;
            bv[u] = dim < d ? __ldg(xb + (size_t)dim * n) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < kPF; ++u)
            if (kb + 4 * u < d4) dmma64(d0, d1, xa[kb + 4 * u], bv[u]);
        }
        const int j0 = 8 * J + 2 * tig;
        double k0v = 0.0, k1v = 0.0;
        // r^2 clamped at 0 by a compare that keeps NaN (fmax(NaN, 0) = 0 would turn a NaN
        // candidate row into a finite one at distance 0)
        auto clamp0 = [](double r2) { return r2 < 0.0 ? 0.0 : r2; };
        if (j0 < n) {
          k0v = kernel64(clamp0(qa + qj[j0] - 2.0 * d0), sf2, m.kernel);
          mu = fma(k0v, __ldg(alpha + j0), mu);
        }
        if (j0 + 1 < n) {
          k1v = kernel64(clamp0(qa + qj[j0 + 1] - 2.0 * d1), sf2, m.kernel);
          mu = fma(k1v, __ldg(alpha + j0 + 1), mu);
        }
        ks[j0 * kPostLd + 8 * cb + gid] = k0v;
        ks[(j0 + 1) * kPostLd + 8 * cb + gid] = k1v;
      }
      mu += __shfl_xor_sync(0xffffffffu, mu, 1);
      mu += __shfl_xor_sync(0xffffffffu, mu, 2);
      if (tig == 0) red[(warp >> 2) * kPostTile + 8 * cb + gid] = mu;  // [kGroups][kPostTile]
    }
    __syncthreads();  // ks complete
    // 3. v = L^-1 k* on DMMA, |v|^2 per candidate
    double vv[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    for (int J = nt - 1; J >= 0; --J) {
      if (owner[J] != warp) continue;
      const int j = 8 * J + gid;
      const double *Lrow = Li + (size_t)min(j, n - 1) * n;
      const int nks = 2 * J + 2;  // k-steps of 4 covering k < 8 J + 8
      // kAcc accumulator sets (k-step parity): 4 kAcc independent DMMA chains per warp
      double acc[kAcc][4][2] = {};
      double an[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = 4 * u + tig;
        an[u] = (u < nks && k <= j && j < n) ? __ldg(Lrow + k) : 0.0;
      }
      for (int k0 = 0; k0 < nks; k0 += 4) {
        double ac[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) ac[u] = an[u];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kk = k0 + 4 + u, k = 4 * kk + tig;
          an[u] = (kk < nks && k <= j && j < n) ? __ldg(Lrow + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kk = k0 + u;
          if (kk < nks) {
            const double *brow = ks + (4 * kk + tig) * kPostLd + gid;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              dmma64(acc[u % kAcc][q][0], acc[u % kAcc][q][1], ac[u], brow[8 * q]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double v0 = acc[0][q][0], v1 = acc[0][q][1];
#pragma unroll
        for (int h = 1; h < kAcc; ++h) { v0 += acc[h][q][0]; v1 += acc[h][q][1]; }
        vv[q][0] = fma(v0, v0, vv[q][0]);
        vv[q][1] = fma(v1, v1, vv[q][1]);
      }
    }
    // rows gid -> one partial per (warp, candidate 8 q + 2 tig + h), fixed shuffle order
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v = vv[q][h];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (gid == 0) red[(kPostWarps + warp) * kPostTile + 8 * q + 2 * tig + h] = v;
      }
    __syncthreads();
    if (tid < cnt) {
      const int c = tid;
      double mu_s = 0.0, vv_s = 0.0;
      for (int q = 0; q < kGroups; ++q) mu_s += red[q * kPostTile + c];
      for (int q = 0; q < kPostWarps; ++q) vv_s += red[(kPostWarps + q) * kPostTile + c];
      const int64_t e = row0 + c;
      const bool fin = isfinite(mu_s) && isfinite(vv_s);  // NaN rows: NaN outputs
      const double var64 = fmax(sf2 - vv_s, 0.0);
      const double sig = sqrt(var64);
      const double imp = best - mu_s;
      const double ei = sig > 0.0 ? sig * tau64(imp / sig) : fmax(imp, 0.0);
      if (p.out_mu) p.out_mu[e] = fin ? (float)(m.mean + m.std * mu_s) : NAN;
      if (p.out_var) p.out_var[e] = fin ? (float)(m.std * m.std * var64) : NAN;
      if (p.out_ei) p.out_ei[e] = fin ? (float)(m.std * ei) : NAN;
    }
  }
}

}  // namespace

template <int W>
static cudaError_t launch_post(const RefineLaunch &p, int n8, int dmax, int num_sms,
                               cudaStream_t stream) {
  const int xld = (dmax + 3) / 4 * 4 + 1;
  const size_t smem = ((size_t)n8 * kPostLd + (size_t)kPostTile * xld + n8 + kPostTile +
                       2 * W * kPostTile) * sizeof(double) + (size_t)(n8 / 8) * sizeof(int);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(posterior64_kernel<W>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, posterior64_kernel<W>, 32 * W, smem);
  const int64_t tiles = (p.dense_rows + kPostTile - 1) / kPostTile;
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)num_sms * std::max(per_sm, 1));
  posterior64_kernel<W><<<grid, 32 * W, smem, stream>>>(p, dmax);
  return cudaGetLastError();
}

cudaError_t launch_posterior64(const RefineLaunch &p, int nmax, int dmax, int num_sms,
                               cudaStream_t stream) {
  if (p.dense_rows <= 0) return cudaSuccess;
  const int n8 = (nmax + 7) / 8 * 8;
  return n8 > 256 ? launch_post<16>(p, n8, dmax, num_sms, stream)
                  : launch_post<GPBO_POST_WSMALL>(p, n8, dmax, num_sms, stream);
}

cudaError_t launch_refine(const RefineLaunch &p, int64_t max_entries, int num_sms, int nmax,
                          cudaStream_t stream) {
  if (max_entries <= 0) return cudaSuccess;
  // argmax mode with long L^-1 rows (n > 128: configs 2, 4): clusters of kSplit CTAs per flagged
  // candidate, 4 CTAs per SM (config 2 refine 23 -> 17 us, config 4 92 -> 41 us).  Small n with
  // many flagged candidates (config 3: ~3.5k) keeps one CTA per candidate (56 vs 371 us).
  if (p.list && nmax > 128) {
    const int kSplit = nmax <= 256 ? 4 : 8;
    const int64_t ncl = std::max<int64_t>(1, std::min<int64_t>(max_entries, num_sms * 4 / kSplit));
    // programmatic dependent launch after the fast phase (griddepcontrol.wait inside); the
    // cluster shape comes from __cluster_dims__
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(ncl * kSplit));
    cfg.blockDim = dim3(kRefineThreads);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return kSplit == 4 ? cudaLaunchKernelEx(&cfg, refine_split_kernel<4>, p)
                       : cudaLaunchKernelEx(&cfg, refine_split_kernel<8>, p);
  }
#ifndef GPBO_REFINE_WARP
#define GPBO_REFINE_WARP 1
#endif
  // a warp per entry for long lists (the list scales with the candidates: >= 2^21 rows means
  // >= 128 audit entries alone; config 3, 2^24 rows: ~5,000 entries, 0.076 -> 0.065 ms), a CTA
  // per entry for short ones, where one entry's latency bounds the phase (config 5, 2^18 rows:
  // ~200 entries, 0.019 ms with CTAs vs 0.029 with warps)
  if (GPBO_REFINE_WARP && p.list && nmax <= 128 && max_entries >= (int64_t(1) << 21)) {
    const int64_t blocks = (max_entries + kRwWarps - 1) / kRwWarps;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)num_sms * 8)));
    cfg.blockDim = dim3(32 * kRwWarps);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, refine_warp_kernel, p);
  }
  const int grid = (int)std::min<int64_t>(max_entries, (int64_t)num_sms * 4);
  refine_kernel<<<grid, kRefineThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_direct(const RefineLaunch &p, int S, int64_t rows, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  direct_kernel<<<(unsigned)((rows + kDirectWarps - 1) / kDirectWarps), 32 * kDirectWarps, 0,
                  stream>>>(p, S, rows);
  return cudaGetLastError();
}

}  // namespace gpbo
