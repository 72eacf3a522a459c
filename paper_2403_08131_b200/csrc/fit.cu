// H1-H4 of the hot path: standardise y, Gram matrix, jittered Cholesky,
// triangular inverse, alpha -- one CTA per sub-search, float64 throughout.
//
// PAPER.md L249/L256 (§IV.D): the GP's "O(N^3) training complexity" is this factorisation.
// The kernel/jitter/standardisation readings are R1, R2, R7, R9 of DESIGN.md.
//
// Layout: the working matrix W is the lower triangle of an n x n float64 matrix stored as the
// lower triangle of 8 x 8 tiles, each tile row-major (= the DMMA accumulator fragment order).
// For n <= kFitSmemMaxN it lives in shared memory (189 KB at n = 216); otherwise in a global
// scratch buffer of the model (L2 resident).
//
// Factorisation (H3) and inversion (H4) are ONE elimination sweep: the row operations that reduce
// K to L^T, applied to I, give L^-1 ([K | I] -> [L^T | L^-1] up to the row scaling).  Both halves
// share one lower triangle W: after step j, W(i, k) holds L^-1 for k <= j and the reduced K for
// k > j.  Step j (pivot p = W(j, j), column c_i = W(i, j), i > j; g = row j left of j and column
// j below it):  W(i, k) -= (c_i / p) g_k for i > j with W(i, j) := -c_i / p;  row j *= 1/sqrt(p);
// L(i, j) = c_i / sqrt(p).  Blocked by kFitB = 8 steps (block [J, J + 8)):
//   D  the 8 x 8 diagonal block, sequentially in one warp (registers + shuffles).  The steps act
//      linearly on any other row's 8 block entries x and on any block column w left of the
//      block, so the same warp also runs them on unit vectors and records three 8 x 8 maps:
//        row i below the block:  L(i, J + u) = (x N)_u,   new W(i, J + k) = (x M)_k
//        column k left of it:    new W(J + t, k) = (R w)_t  (= L^-1(J + t, k), final)
//   C  those two products for all rows below / columns left of the block on the FP64 tensor
//      cores (DMMA m8n8k4); the L panel and the final block rows of L^-1 go to G[u][.];
//   T  the rest: W(i, k) -= sum_u G[u][i] G[u][k] over rows below the block x (columns left of
//      it and the trailing triangle), 8 x 8 DMMA tiles dealt to the warps.  Warp 0 updates the
//      next diagonal block first and runs its D while the other warps finish T (look-ahead).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>

#include "gpbo_internal.cuh"
#include "score_pack.cuh"

namespace gpbo {
namespace {

constexpr int kWarps = kFitThreads / 32;
#ifndef GPBO_FIT_QW
#define GPBO_FIT_QW 4
#endif
constexpr int kQ = GPBO_FIT_QW;  // tiles of one tile row per trailing-update work item (<= kQ)
#ifndef GPBO_FIT_STATIC
#define GPBO_FIT_STATIC 1  // T work list: static 4-aligned quads (1) or per-row items (0)
#endif
static_assert(kFitB == 8, "the DMMA tiling of fit.cu assumes 8-step panels");

#ifdef GPBO_FIT_TIMING  // phase clocks of CTA 0 printed at exit (tools/fit_phases.py)
#define FIT_T(slot) do { if (blockIdx.x == 0 && threadIdx.x == 0) fit_t[slot] += clock64() - fit_t0; fit_t0 = clock64(); } while (0)
#else
#define FIT_T(slot) do { } while (0)
#endif

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

// 1 / sqrt(p): the MUFU approximation refined by two Newton steps (quadratic convergence from
// ~2^-22 to the float64 rounding level) -- short latency, no special-case branches (a failed
// pivot is flagged by the caller and its values discarded).
__device__ __forceinline__ double rsqrt_fast(double p) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(p));
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double e = fma(-p, y * y, 1.0);
    y = fma(0.5 * y, e, y);
  }
  return y;
}

__device__ __forceinline__ double kernel_value(double r2, double sf2, int kind) {
  if (kind == GPBO_RBF) return sf2 * exp(-0.5 * r2);
  const double r = sqrt(r2);
  const double s5 = 2.23606797749978969640917366873;  // sqrt(5)
  return sf2 * (1.0 + s5 * r + (5.0 / 3.0) * r2) * exp(-s5 * r);
}

// D = A B + D on the FP64 tensor cores, m8n8k4: lane l holds A[l/4][l%4], B[l%4][l/4] and
// D[l/4][2 (l%4)], D[l/4][2 (l%4) + 1].
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// Tile (R, C), C <= R, of the tile-packed lower triangle: 64 doubles, row-major.  The
// row-major 8 x 8 order IS the DMMA accumulator fragment order (lane l holds elements 2l and
// 2l + 1), so accumulator tiles move with one 16-byte access per lane.
__device__ __forceinline__ int tb(int R, int C) { return (R * (R + 1) / 2 + C) * 64; }

// Tile index e -> (R, C) of the lower triangle, row-major.
__device__ __forceinline__ void tile_rc(int e, int &R, int &C) {
  R = (int)((sqrtf(8.f * e + 1.f) - 1.f) * 0.5f);
  while ((R + 1) * (R + 2) / 2 <= e) ++R;
  while (R * (R + 1) / 2 > e) --R;
  C = e - R * (R + 1) / 2;
}

// The body is instantiated for a shared-memory and a global working matrix so that every access
// to W compiles to LDS/STS or LDG/STG instead of generic loads.
template <bool kSmem>
__device__ __forceinline__ void fit_body(double *sm, double *red,
                                         const SearchMeta *__restrict__ meta_in, const FitIO &io,
                                         SearchMeta *__restrict__ meta_out) {
  double *L64 = io.L64, *Linv64 = io.Linv64, *Xs64 = io.Xs64, *alpha64 = io.alpha64;
  double *Wscr64 = io.Wscr64;
  const int s = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;  // DMMA fragment coordinates
  SearchMeta m = meta_in[s];
  if (io.sf2_src) { m.sf2 = io.sf2_src[s]; m.sn2 = io.sn2_src[s]; }
  const int n = m.n, d = m.d;
#ifdef GPBO_FIT_TIMING
  long long fit_t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long fit_t0 = clock64();
  long long fit_tw = 0, fit_tD = 0;
#endif
  const int nr8 = fit_nr8(n), gs = fit_gstride(n), nt = (n + 7) / 8;
  double *yt = sm;                     // y~ (n)
  double *w = sm + nr8;                // L^-1 y~ (n)
  double *piv = sm + 2 * nr8;          // [16]: the last D's fail flag (rest spare)
  double *Mm = piv + 24;               // the block maps M, N, R (8 x 8 each, row-major)
  double *Nm = Mm + 64;
  double *Rm = Nm + 64;
  double *G = Rm + 64;                 // G[u][.], 2 x 8 rows of gs (a pair of panels)
  double *W = kSmem ? G + 16 * gs : Wscr64 + m.scr_off;
  // element (i, k), i >= k
  auto at = [&](int i, int k) -> int { return tb(i >> 3, k >> 3) + 8 * (i & 7) + (k & 7); };
  double *Lg = L64 + m.mat_off;        // L, col-major (lower part; export zeroes the rest)
  const float *X = io.X_src + m.x_off;
  const float *ls = io.ls_src + m.ls_off;
  const double *y = io.y_src + m.y_off;

  // ---- input validation (GPBO_EINVAL on any non-finite / out-of-domain value), copying the
  // inputs into the model when they come from the caller's device arrays
  const bool copy = io.X_src != io.X32;
  int bad = 0;
  for (int i = tid; i < n * d; i += kFitThreads) bad |= !isfinite(X[i]);  // (copied by the pre-pass)
  for (int i = tid; i < n; i += kFitThreads) {
    bad |= !isfinite(y[i]);
    if (copy) io.y64[m.y_off + i] = y[i];
  }
  for (int i = tid; i < d; i += kFitThreads) {
    bad |= !(ls[i] > 0.f) || !isfinite(ls[i]);
    if (copy) io.ls32[m.ls_off + i] = ls[i];
  }
  bad |= !(m.sf2 > 0.f) || !isfinite(m.sf2) || !(m.sn2 >= 0.f) || !isfinite(m.sn2);
  bad = __syncthreads_or(bad);
  if (bad) {
    if (tid == 0) { m.status = GPBO_EINVAL; m.jitter_k = -1; m.lml = -INFINITY; meta_out[s] = m; }
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

  // Programmatic dependent launch: everything above reads only the caller's inputs and ran
  // while the Gram pre-pass was still executing; from here on its outputs are read.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // ---- pmax = max_j |x_j / l|^2 (the pre-pass's per-CTA maxima)
  double pmax = 0.0;
  for (int b = 0; b * 128 < n; ++b) pmax = fmax(pmax, io.pm_part[16 * s + b]);

  // ---- H2 + H3 + H4 along the jitter ladder j_k = 1e-8 10^k sf2
  const double sf2 = m.sf2, sn2 = m.sn2;
  const double *xc = Xs64 + m.x_off;
  const int ntiles = nt * (nt + 1) / 2;

  // D (warp 0): the diagonal block A11 = W[J..J+8, J..J+8) (padded with identity rows for a
  // ragged last block).  Lane 0 factors it in registers, L11 = chol(A11) and X = L11^-1 (in
  // place, column by column); then the warp forms the maps C applies (see the header):
  //   N = X^T  (L21 = A21 L11^-T),  M = -X^T X  (= -A11^-1),  R = X.
  // The diagonal block of W becomes X (its final L^-1 entries); piv[16] flags a pivot <= 0.
  auto diag_block = [&](int J) {
    const int bb = min(kFitB, n - J);
    double *Wd = W + tb(J >> 3, J >> 3);
    if (lane == 0) {
      double a[36];  // packed lower, row-major: (i, k) at i (i + 1) / 2 + k
      double rr[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int k = 0; k <= i; ++k)
          a[i * (i + 1) / 2 + k] = i < bb ? Wd[8 * i + k] : (i == k ? 1.0 : 0.0);
      bool fail = false;
#pragma unroll
      for (int j = 0; j < 8; ++j) {  // right-looking Cholesky
        const double p = a[j * (j + 1) / 2 + j];
        fail |= !(p > 0.0) || !isfinite(p);
        const double r = rsqrt_fast(p);
        rr[j] = r;
        a[j * (j + 1) / 2 + j] = p * r;
#pragma unroll
        for (int i = j + 1; i < 8; ++i) a[i * (i + 1) / 2 + j] *= r;
#pragma unroll
        for (int i = j + 1; i < 8; ++i)
#pragma unroll
          for (int k = j + 1; k <= i; ++k)
            a[i * (i + 1) / 2 + k] = fma(-a[i * (i + 1) / 2 + j], a[k * (k + 1) / 2 + j],
                                         a[i * (i + 1) / 2 + k]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)  // L11 -> Nm (scratch until the maps are formed)
#pragma unroll
        for (int k = 0; k <= i; ++k) Nm[8 * i + k] = a[i * (i + 1) / 2 + k];
#pragma unroll
      for (int j = 0; j < 8; ++j) {  // X = L^-1 in place: X_ij = -r_i sum_{k=j}^{i-1} L_ik X_kj
        a[j * (j + 1) / 2 + j] = rr[j];
#pragma unroll
        for (int i = j + 1; i < 8; ++i) {
          double t = 0.0;
#pragma unroll
          for (int k = j; k < i; ++k) t = fma(a[i * (i + 1) / 2 + k], a[k * (k + 1) / 2 + j], t);
          a[i * (i + 1) / 2 + j] = -rr[i] * t;
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)  // X -> Rm (lower part)
#pragma unroll
        for (int k = 0; k <= i; ++k) Rm[8 * i + k] = a[i * (i + 1) / 2 + k];
      piv[16] = fail ? 1.0 : 0.0;
    }
    __syncwarp();
    // the warp spreads the outputs: L11 to L64, X to the diagonal tile, R = X, N = X^T
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h, i = e >> 3, k = e & 7;
      if (k <= i && i < bb) Lg[(size_t)(J + k) * n + J + i] = Nm[e];
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h, i = e >> 3, k = e & 7;
      const double v = k <= i ? Rm[e] : 0.0;
      Wd[e] = v;
      Nm[8 * k + i] = v;
      if (k > i) Rm[e] = 0.0;
    }
    __syncwarp();
    // M = -X^T X: lane -> entries (mr, mc) = (e / 8, e % 8), e = lane, lane + 32
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h, mr = e >> 3, mc = e & 7;
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) t = fma(Rm[q * 8 + mr], Rm[q * 8 + mc], t);
      Mm[e] = -t;
    }
  };

  int jk = -1;
  double jit = 0.0;
  double p10 = 1.0;
#if GPBO_FIT_STATIC
  static_assert(kQ == 4, "the static quad list assumes 4-tile quads");
  // the trailing update's quad list: (R, Q) for rows R = nt - 1 .. 1, Q = 0 .. R / kQ;
  // qabove[J] = number of quads of rows > J
  __shared__ int qtab[(kFitSmemMaxN / 8) * (kFitSmemMaxN / 8 / kQ + 1)];
  __shared__ int qabove[kFitSmemMaxN / 8 + 1];
  if (kSmem && tid == 0) {
    int k = 0;
    for (int R = nt - 1; R >= 1; --R) {
      for (int Q = 0; Q <= R / kQ; ++Q) qtab[k++] = R << 8 | Q;
      qabove[R - 1] = k;
    }
  }
#endif
  FIT_T(0);
  for (int k = 0; k < 7 && jk < 0; ++k, p10 *= 10.0) {
    jit = 1e-8 * p10 * sf2;
    __syncthreads();
    // H2: the pre-pass's kernel tiles (L2) into W, 4 x 16 B in flight per thread, then + sn2 +
    // jitter on the diagonal
    {
      const double2 *src = reinterpret_cast<const double2 *>(io.Kt64 + m.kt_off);
      double2 *dst = reinterpret_cast<double2 *>(W);
      const int n2 = ntiles * 32;
      for (int e0 = tid; e0 < n2; e0 += 4 * kFitThreads) {
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e0 + u * kFitThreads < n2) v[u] = src[e0 + u * kFitThreads];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e0 + u * kFitThreads < n2) dst[e0 + u * kFitThreads] = v[u];
      }
      __syncthreads();
      for (int i = tid; i < n; i += kFitThreads) W[at(i, i)] += sn2 + jit;
    }
    __syncthreads();
    FIT_T(1);
    if (warp == kWarps - 1) diag_block(0);
    __syncthreads();
    FIT_T(2);
    bool ok = piv[16] == 0.0;
    // Global working matrix: panels are processed in pairs (blocks JT, JT + 1) so the bulk of the
    // trailing update is ONE
    // pass over W with K = 16 (both panels' G), halving the W tile traffic (the T phase is
    // shared-memory bound):
    //   C(JT)  -> G1;  partial T: G1 into tile column JT + 1 (rows below it) and tile row JT + 1
    //   (columns left of JT) -- exactly what D(JT + 1) and C(JT + 1) read; the D warp updates the
    //   diagonal tile JT + 1 and runs D(JT + 1) meanwhile;
    //   C(JT + 1) -> G2;  combined T over rows R > JT + 1: columns C < JT and JT + 1 < C <= R get
    //   G1 and G2, column JT gets G2 only (G1 skips its own block column), column JT + 1 nothing
    //   more (G1 was applied, G2 skips it); the D warp updates diagonal tile JT + 2 and runs D.
    // A ragged single last block has no trailing update.
    double *G1 = G, *G2 = G + 8 * gs;
    // -- C: rows below block JT (tile rows R > JT: [x N | x M]) and columns left of it (tile
    // columns C < JT: R w), on DMMA; the block's G rows go to Gc
    auto cphase = [&](int JT, double *Gc) {
      const int J = 8 * JT, bb = min(kFitB, n - J);
      const int nrt = nt - JT - 1;
      // the maps' fragments are the same for every item of the panel: loaded once
      double nf[2], mf[2], rf[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kk = 4 * h;
        nf[h] = Nm[(kk + tig) * 8 + gid];
        mf[h] = Mm[(kk + tig) * 8 + gid];
        rf[h] = Rm[gid * 8 + kk + tig];
      }
      for (int it = warp; it < nrt + JT; it += kWarps) {
        double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
        if (it < nrt) {
          const int R = JT + 1 + it, i = 8 * R + gid;
          double *Wt = W + tb(R, JT);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double a = Wt[8 * gid + 4 * h + tig];
            dmma(d0, d1, a, nf[h]);
            dmma(e0, e1, a, mf[h]);
          }
          const int u = 2 * tig;
          Gc[u * gs + i] = d0;
          Gc[(u + 1) * gs + i] = d1;
          if (i < n) {
            Lg[(size_t)(J + u) * n + i] = d0;
            Lg[(size_t)(J + u + 1) * n + i] = d1;
          }
          __syncwarp();  // every lane's tile reads precede the write-back (racecheck-clean)
          *reinterpret_cast<double2 *>(Wt + 2 * lane) = make_double2(e0, e1);
        } else {
          const int C = it - nrt;
          double *Wt = W + tb(JT, C);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int mrow = 4 * h + tig;
            const double b = mrow < bb ? Wt[8 * mrow + gid] : 0.0;
            dmma(d0, d1, rf[h], b);
          }
          const int kc = 8 * C + 2 * tig;
          Gc[gid * gs + kc] = d0;
          Gc[gid * gs + kc + 1] = d1;
          __syncwarp();
          *reinterpret_cast<double2 *>(Wt + 2 * lane) = make_double2(d0, d1);
        }
      }
    };
    // W(R, C0 + q) -= sum over the given G buffers of G[u][i] G[u][k], q < cnt (<= 4 tiles of
    // one tile row sharing the A fragments); nb = 1 (Ga) or 2 (Ga and Gb, K = 16)
    auto quad = [&](const double *Ga, const double *Gb, int R, int C0, int cnt) {
      const int i = 8 * R + gid;
      double *Wt = W + tb(R, C0) + 2 * lane;
      double2 c[kQ];
#pragma unroll
      for (int q = 0; q < kQ; ++q)
        if (q < cnt) c[q] = *reinterpret_cast<const double2 *>(Wt + 64 * q);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double *Gh = h == 0 ? Ga : Gb;
        if (Gh == nullptr) continue;
        const double a0 = -Gh[tig * gs + i], a1 = -Gh[(4 + tig) * gs + i];
        const double *g0 = Gh + tig * gs + 8 * C0 + gid, *g1 = g0 + 4 * gs;
        double b0[kQ], b1[kQ];
#pragma unroll
        for (int q = 0; q < kQ; ++q)
          if (q < cnt) { b0[q] = g0[8 * q]; b1[q] = g1[8 * q]; }
#pragma unroll
        for (int q = 0; q < kQ; ++q)
          if (q < cnt) dmma(c[q].x, c[q].y, a0, b0[q]);
#pragma unroll
        for (int q = 0; q < kQ; ++q)
          if (q < cnt) dmma(c[q].x, c[q].y, a1, b1[q]);
      }
#pragma unroll
      for (int q = 0; q < kQ; ++q)
        if (q < cnt) *reinterpret_cast<double2 *>(Wt + 64 * q) = c[q];
    };
    // quad() for one G buffer and a full quad (kQ tiles): no per-tile predicates (a predicated
    // mma.sync costs a WARPSYNC + NOP pair per DMMA) and one base address per operand stream
    // (the predicated form rematerialised every address: ~3x the instructions per tile)
    auto quad_full = [&](const double *__restrict__ Ga, int R, int C0) {
      double *Wt = W + tb(R, C0) + 2 * lane;
      const double *ga = Ga + tig * gs + 8 * R + gid;
      const double *gb = Ga + tig * gs + 8 * C0 + gid;
      double2 c[kQ];
#pragma unroll
      for (int q = 0; q < kQ; ++q) c[q] = *reinterpret_cast<const double2 *>(Wt + 64 * q);
      const double a0 = -ga[0], a1 = -ga[4 * gs];
      double b0[kQ], b1[kQ];
#pragma unroll
      for (int q = 0; q < kQ; ++q) { b0[q] = gb[8 * q]; b1[q] = gb[4 * gs + 8 * q]; }
#pragma unroll
      for (int q = 0; q < kQ; ++q) dmma(c[q].x, c[q].y, a0, b0[q]);
#pragma unroll
      for (int q = 0; q < kQ; ++q) dmma(c[q].x, c[q].y, a1, b1[q]);
#pragma unroll
      for (int q = 0; q < kQ; ++q) *reinterpret_cast<double2 *>(Wt + 64 * q) = c[q];
    };
    // quad() over the tiles of a 4-aligned quad selected by `mask` (one G buffer)
    auto quad_mask = [&](const double *Ga, int R, int C0, unsigned mask) {
      double *Wt = W + tb(R, C0) + 2 * lane;
      const double *ga = Ga + tig * gs + 8 * R + gid;
      const double *gb = Ga + tig * gs + 8 * C0 + gid;
      double2 c[kQ];
#pragma unroll
      for (int q = 0; q < kQ; ++q)
        if (mask >> q & 1) c[q] = *reinterpret_cast<const double2 *>(Wt + 64 * q);
      const double a0 = -ga[0], a1 = -ga[4 * gs];
#pragma unroll
      for (int q = 0; q < kQ; ++q)
        if (mask >> q & 1) {
          dmma(c[q].x, c[q].y, a0, gb[8 * q]);
          dmma(c[q].x, c[q].y, a1, gb[4 * gs + 8 * q]);
          *reinterpret_cast<double2 *>(Wt + 64 * q) = c[q];
        }
    };
    constexpr int kT = kWarps - 1;  // T warps (the highest warp is the D warp)
    // The working matrix in shared memory: one panel per step, the trailing update overlapping
    // the next block's D (D's latency is hidden behind a full T pass; measured faster than
    // pairs at n = 200).  In global memory (n > kFitSmemMaxN, L2 traffic bound): pairs.
    for (int JT = 0; kSmem && JT < nt && ok; ++JT) {
      cphase(JT, G1);
      __syncthreads();
      FIT_T(3);
      if (JT + 1 == nt) break;
      const int nrt = nt - JT - 1, nlq = (JT + kQ - 1) / kQ;
      if (warp == kWarps - 1) {  // look-ahead: the next diagonal tile, then its D
        quad(G1, nullptr, JT + 1, JT + 1, 1);
        __syncwarp();
        diag_block(8 * (JT + 1));
      } else {
#if GPBO_FIT_STATIC
        // 4-aligned quads (R, Q) of the rows below the panel, rows descending (qtab): the quads
        // of rows > JT are the first qabove[JT] entries, dealt round robin; a quad's tiles at
        // the panel column JT, past the diagonal, or on the D warp's diagonal tile are masked
        const int nq = qabove[JT];
        // tiles of quad (R, C0) to update: C <= R, not the panel column JT, not the D warp's
        // diagonal tile (R = JT + 1)
        auto qmask = [&](int R, int C0) -> unsigned {
          unsigned mk = 0xFu;
          if (C0 + 3 > R) mk &= (1u << (R - C0 + 1)) - 1u;
          if (JT >= C0 && JT < C0 + 4) mk &= ~(1u << (JT - C0));
          if (R == JT + 1 && R < C0 + 4) mk &= ~(1u << (R - C0));
          return mk;
        };
        for (int k = warp; k < nq; k += kT) {
          const int v = qtab[k], R = v >> 8, C0 = kQ * (v & 255);
          const unsigned mask = qmask(R, C0);
          if (mask == 0xFu) quad_full(G1, R, C0);
          else if (mask) quad_mask(G1, R, C0, mask);
        }
#else
        // items of tile row r (R = JT + 1 + r): nlq left quads, then r / 4 + 1 right quads
        // (row 0's right quad is the diagonal tile -- the D warp's), round robin, rotated
        for (int r = 0, w0 = 0; r < nrt; ++r, w0 = (w0 + 5) % kT) {
          const int R = JT + 1 + r, len = nlq + (r > 0 ? r / kQ + 1 : 0);
          for (int q = (warp - w0 + kT) % kT; q < len; q += kT) {
            int C0, cnt;
            if (q < nlq) {
              C0 = kQ * q;
              cnt = min(kQ, JT - kQ * q);
            } else {
              const int c0 = kQ * (q - nlq);
              C0 = JT + 1 + c0;
              cnt = min(kQ, r + 1 - c0);
            }
            if (cnt == kQ) quad_full(G1, R, C0);
            else quad(G1, nullptr, R, C0, cnt);
          }
        }
#endif
      }
      __syncthreads();
      FIT_T(4);
      ok = piv[16] == 0.0;  // the next block's D (uniform)
    }
    for (int JT = 0; !kSmem && JT < nt && ok;) {
      const bool pair = JT + 1 < nt;
      cphase(JT, G1);
      __syncthreads();
      FIT_T(3);
      if (!pair) { ++JT; break; }
      // -- partial T(JT) with G1: tile column JT + 1 below its diagonal, tile row JT + 1 left of
      // JT; the D warp: the diagonal tile JT + 1, then D(JT + 1)
      {
        const int nlq = (JT + 3) / 4, ncol = nt - JT - 2;
        if (warp == kWarps - 1) {
          quad(G1, nullptr, JT + 1, JT + 1, 1);
          __syncwarp();
          diag_block(8 * (JT + 1));
        } else {
          for (int q = warp; q < ncol + nlq; q += kT) {
            if (q < ncol) quad(G1, nullptr, JT + 2 + q, JT + 1, 1);
            else quad(G1, nullptr, JT + 1, 4 * (q - ncol), min(4, JT - 4 * (q - ncol)));
          }
        }
      }
      __syncthreads();
      FIT_T(4);
      ok = piv[16] == 0.0;
      if (!ok) break;
      cphase(JT + 1, G2);
      __syncthreads();
      FIT_T(3);
      // -- combined T over tile rows R > JT + 1
      const int R0 = JT + 2;
      if (R0 < nt) {
        const int nrt = nt - R0, nlq = (JT + 3) / 4;
        if (warp == kWarps - 1) {  // look-ahead: the next diagonal tile, then its D
          quad(G1, G2, R0, R0, 1);
          __syncwarp();
#ifdef GPBO_FIT_TIMING
          const long long td0 = clock64();
#endif
          diag_block(8 * R0);
#ifdef GPBO_FIT_TIMING
          if (blockIdx.x == 0 && lane == 0) fit_tD += clock64() - td0;
#endif
        } else {
#ifdef GPBO_FIT_TIMING
          const long long tw0 = clock64();
#endif
          // items of tile row r (R = R0 + r): nlq left quads (G1 + G2), the column-JT tile
          // (G2 only), then r / 4 + 1 right quads from column R0 (row 0's is the diagonal tile:
          // the D warp's).  Round robin over the T warps, rotated per row.
          for (int r = 0, w0 = 0; r < nrt; ++r, w0 = (w0 + 5) % kT) {
            const int R = R0 + r, len = nlq + 1 + (r >> 2) + (r > 0 ? 1 : 0);
            for (int q = (warp - w0 + kT) % kT; q < len; q += kT) {
              if (q < nlq) {
                quad(G1, G2, R, 4 * q, min(4, JT - 4 * q));
              } else if (q == nlq) {
                quad(G2, nullptr, R, JT, 1);
              } else {
                const int c0 = 4 * (q - nlq - 1);
                quad(G1, G2, R, R0 + c0, min(4, r + 1 - c0));
              }
            }
          }
#ifdef GPBO_FIT_TIMING
          if (blockIdx.x == 0 && threadIdx.x == 0) fit_tw += clock64() - tw0;
#endif
        }
        __syncthreads();
        FIT_T(4);
        ok = piv[16] == 0.0;  // the next block's D (uniform)
      }
      JT += 2;
    }
    if (ok) jk = k;
  }
  __syncthreads();
  if (jk < 0) {
    if (tid == 0) {
      m.status = GPBO_ENOTPD; m.jitter_k = -1; m.jitter = NAN; m.lml = -INFINITY;
      m.mean = mean; m.std = stdv; m.best = best; m.alpha_l1 = 0.0;
      meta_out[s] = m;
    }
    return;
  }
  // ---- W now holds L^-1 (lower).  w = L^-1 y~ with the row abs sums and the abs max: warp
  // per tile row, lane -> row gid of the tile, columns 2 tig + {0, 1} (one 16-byte load per lane
  // and tile); the tiles go to the row-major L^-1 on the way (the refine phase, the tcgen05
  // image and the CUDA-core operands read only k <= i).
  // (ld = sum_i log L_ii = -sum_i log (L^-1)_ii and ww = |w|^2 = y~^T alpha feed the log marginal
  // likelihood, §8(f)1 ML-II)
  double rs = 0.0, lam = 0.0, ld = 0.0, ww = 0.0;
  for (int R = warp; R < nt; R += kWarps) {
    const int i = 8 * R + gid;
    double a2 = 0.0, a3 = 0.0;
    double *dst = Linv64 + m.mat_off + (size_t)min(i, n - 1) * n;
    for (int C = 0; C <= R; ++C) {
      const double2 v = *reinterpret_cast<const double2 *>(W + tb(R, C) + 2 * lane);
      const int c0 = 8 * C + 2 * tig;
      const bool in0 = i < n && c0 <= i, in1 = i < n && c0 + 1 <= i;
      const double v0 = in0 ? v.x : 0.0, v1 = in1 ? v.y : 0.0;
      a2 = fma(v0, yt[min(c0, n - 1)], a2);
      a2 = fma(v1, yt[min(c0 + 1, n - 1)], a2);
      a3 += fabs(v0) + fabs(v1);
      lam = fmax(lam, fmax(fabs(v0), fabs(v1)));
      if (in0) dst[c0] = v.x;
      if (in1) dst[c0 + 1] = v.y;
      if (in0 && c0 == i) ld -= log(v.x);
      if (in1 && c0 + 1 == i) ld -= log(v.y);
    }
    a2 += __shfl_xor_sync(0xffffffffu, a2, 1);
    a2 += __shfl_xor_sync(0xffffffffu, a2, 2);
    a3 += __shfl_xor_sync(0xffffffffu, a3, 1);
    a3 += __shfl_xor_sync(0xffffffffu, a3, 2);
    if (tig == 0 && i < n) {
      w[i] = a2;
      ww = fma(a2, a2, ww);
    }
    rs = fmax(rs, a3);
  }
  __syncthreads();
  // alpha = L^-T w: warp per tile column, lane -> column pair 2 tig, rows gid of the tiles below
  double l1 = 0.0, amx = 0.0;
  for (int C = warp; C < nt; C += kWarps) {
    const int c0 = 8 * C + 2 * tig;
    double s0 = 0.0, s1 = 0.0;
    for (int R = C; R < nt; ++R) {
      const int i = 8 * R + gid;
      if (i < n) {
        const double2 v = *reinterpret_cast<const double2 *>(W + tb(R, C) + 2 * lane);
        const double wi = w[i];
        if (c0 <= i) s0 = fma(v.x, wi, s0);
        if (c0 + 1 <= i) s1 = fma(v.y, wi, s1);
      }
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (gid == 0) {
      if (c0 < n) {
        alpha64[m.a_off + c0] = s0;
        l1 += fabs(s0);
        amx = fmax(amx, fabs(s0));
      }
      if (c0 + 1 < n) {
        alpha64[m.a_off + c0 + 1] = s1;
        l1 += fabs(s1);
        amx = fmax(amx, fabs(s1));
      }
    }
  }
  for (int kk = n + tid; kk < m.n_pad; kk += kFitThreads) alpha64[m.a_off + kk] = 0.0;
  // the six statistics in one block reduction (sums: l1, ld, ww; maxima: amx, rs, lam), in a
  // fixed order (deterministic)
  {
    double v[6] = {l1, ld, ww, amx, rs, lam};
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, v[q], o);
        v[q] = q < 3 ? v[q] + t : fmax(v[q], t);
      }
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 6; ++q) red[6 * warp + q] = v[q];
    __syncthreads();
    if (tid < 6) {
      double t = red[tid];
      for (int w2 = 1; w2 < kWarps; ++w2) t = tid < 3 ? t + red[6 * w2 + tid] : fmax(t, red[6 * w2 + tid]);
      red[6 * kWarps + tid] = t;
    }
    __syncthreads();
    l1 = red[6 * kWarps];
    ld = red[6 * kWarps + 1];
    ww = red[6 * kWarps + 2];
    amx = red[6 * kWarps + 3];
    rs = red[6 * kWarps + 4];
    lam = red[6 * kWarps + 5];
  }
  FIT_T(5);
#ifdef GPBO_FIT_TIMING
  if (blockIdx.x == 0 && tid == 0)
    printf("FIT_PHASES n=%d setup=%lld gram=%lld diag0=%lld panelC=%lld trailingT=%lld tail=%lld"
           " [warp0 T tiles: %lld]\n", n, fit_t[0], fit_t[1], fit_t[2], fit_t[3], fit_t[4],
           fit_t[5], fit_tw);
  if (blockIdx.x == 0 && tid == kFitThreads - 32) printf("FIT_PHASES D in T: %lld\n", fit_tD);
#endif
  if (tid == 0) {
    m.status = degenerate ? GPBO_WDEGENERATE : GPBO_OK;
    m.jitter_k = jk; m.jitter = jit;
    m.mean = mean; m.std = stdv; m.best = best; m.alpha_l1 = l1;
    m.pmax = (float)pmax; m.alpha_max = (float)amx; m.linv_rowsum = (float)rs;
    m.linv_absmax = lam;
    // log marginal likelihood of y~ at this theta (the jittered K actually factored):
    // -1/2 y~^T alpha - sum_i log L_ii - n/2 log 2 pi  (Rasmussen & Williams eq. 2.30)
    m.lml = -0.5 * ww - ld - 0.5 * n * 1.8378770664093454836;
    m.mean_tier = (double)m.sf2 * l1 > kMeanTierL1 ? 1 : 0;
    meta_out[s] = m;
  }
  // the tcgen05 operand image while L^-1, alpha and x / l are hot (saves the pack launch; small
  // problems, n <= kDirectMaxN, are scored by the float64 direct kernel and need no image)
  if (io.img != nullptr && n > kDirectMaxN && kSmem) {
    __syncthreads();  // meta_out[s], L^-1 (row-major) and alpha written by this block
    const SearchMeta mf = meta_out[s];
    pack_body(meta_out + s, mf, io.Linv64, io.Xs64, io.alpha64, io.ls32, io.img, tid, kFitThreads,
              true, sm, sm + 8);  // (the working matrix's space is free now)
  }
}

// ---- Gram pre-pass (H2), spread over many CTAs so the single-CTA factorisation starts from a
// ready kernel matrix.  One launch, CTA (x, s) of 128 threads:
//   x < ceil(n / 128): x / l in float64 (the oracle's A / l) for points 128 x .. into Xs64
//      (column-major d x n), and the CTA's max |x / l|^2 into pm_part[16 s + x];
//   warp w: tile e = 4 x + w of the tile-packed lower triangle -- its 16 points' x / l staged in
//      shared memory, squared distances by direct differences (reading R1), the kernel (no noise,
//      no jitter: the fit adds them per jitter-ladder step); entries outside the matrix are 0.
__global__ void __launch_bounds__(128)
gram_kernel(const SearchMeta *__restrict__ meta, const FitIO io) {
  __shared__ double xw[4][16][GPBO_MAX_D + 1];
  __shared__ double red[4];
  // let the dependent fit kernel start its input validation / standardisation now; it waits
  // (griddepcontrol.wait) for this grid's completion before reading Xs64 / Kt64 / pm_part
  asm volatile("griddepcontrol.launch_dependents;");
  const int s = blockIdx.y;
  const SearchMeta m = meta[s];
  const int n = m.n, d = m.d, nt = (n + 7) / 8;
  const float *X = io.X_src + m.x_off;
  const float *ls = io.ls_src + m.ls_off;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if ((int)blockIdx.x * 128 < n) {
    const int i = blockIdx.x * 128 + threadIdx.x;
    // the caller's device X is copied into the model here (not in the fit kernel): X32 is then
    // complete when this grid is, and bo_suggest_batch's generator can start on another stream
    // while the factorisation runs (api.cu xready_ev)
    const bool copy = io.X_src != io.X32;
    double q = 0.0;
    if (i < n)
      for (int c = 0; c < d; ++c) {
        const float xv = X[i * d + c];
        if (copy) io.X32[m.x_off + i * d + c] = xv;
        const double v = (double)xv / (double)ls[c];
        io.Xs64[m.x_off + (size_t)c * n + i] = v;
        q += v * v;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q = fmax(q, __shfl_xor_sync(0xffffffffu, q, o));
    if (lane == 0) red[w] = q;
    __syncthreads();
    if (threadIdx.x == 0)
      io.pm_part[16 * s + blockIdx.x] = fmax(fmax(red[0], red[1]), fmax(red[2], red[3]));
  }
  const int e = blockIdx.x * 4 + w;
  if (e >= nt * (nt + 1) / 2) return;
  const int gid = lane >> 2, tig = lane & 3;
  int R, C;
  tile_rc(e, R, C);
  // stage x / l of rows 8R.. (slots 0-7) and columns 8C.. (slots 8-15), clamped to n - 1
  for (int t = lane; t < 16 * d; t += 32) {
    const int slot = t / d, c = t - slot * d;
    const int pt = min((slot < 8 ? 8 * R + slot : 8 * C + slot - 8), n - 1);
    xw[w][slot][c] = (double)X[pt * d + c] / (double)ls[c];
  }
  __syncwarp();
  const int i = 8 * R + gid, kc = 8 * C + 2 * tig;
  const double *xi = xw[w][gid], *xk0 = xw[w][8 + 2 * tig], *xk1 = xw[w][9 + 2 * tig];
  double r0 = 0.0, r1 = 0.0;
  for (int c = 0; c < d; ++c) {
    const double d0 = xi[c] - xk0[c], d1 = xi[c] - xk1[c];
    r0 = fma(d0, d0, r0);
    r1 = fma(d1, d1, r1);
  }
  const double sf2 = io.sf2_src ? (double)io.sf2_src[s] : (double)m.sf2;
  double v0 = 0.0, v1 = 0.0;
  if (i < n && kc <= i) v0 = kernel_value(r0, sf2, m.kernel);
  if (i < n && kc + 1 <= i) v1 = kernel_value(r1, sf2, m.kernel);
  reinterpret_cast<double2 *>(io.Kt64 + m.kt_off + tb(R, C))[lane] = make_double2(v0, v1);
}

__global__ void __launch_bounds__(kFitThreads, 1)
fit_kernel(const SearchMeta *__restrict__ meta_in, const FitIO io,
           SearchMeta *__restrict__ meta_out) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[6 * kWarps + 6];
  if (meta_in[blockIdx.x].use_smem)
    fit_body<true>(sm, red, meta_in, io, meta_out);
  else
    fit_body<false>(sm, red, meta_in, io, meta_out);
}

// CUDA-core scoring operands, built on first use of that path (score_simt.cu): X / l in float32
// (IEEE division of the float32 inputs), zero padded to n_pad x d_pad, and the float32
// (L^-1)^T, LT[k][j] = Linv[j][k] for j >= k, n_pad x n_pad.
__global__ void __launch_bounds__(256)
simt_operands_kernel(const SearchMeta *__restrict__ meta, const float *__restrict__ X32,
                     const float *__restrict__ ls32, const double *__restrict__ Linv64,
                     float *Xs32, float *LT32) {
  const SearchMeta m = meta[blockIdx.x];
  if (m.status != GPBO_OK && m.status != GPBO_WDEGENERATE) return;
  const int n = m.n, d = m.d;
  for (int e = threadIdx.x; e < m.n_pad * m.d_pad; e += blockDim.x) {
    const int i = e / m.d_pad, c = e - i * m.d_pad;
    Xs32[m.xs_off + e] = (i < n && c < d)
                             ? __fdiv_rn(X32[m.x_off + i * d + c], ls32[m.ls_off + c]) : 0.f;
  }
  const double *Li = Linv64 + m.mat_off;
  for (int k = threadIdx.x >> 5; k < m.n_pad; k += blockDim.x >> 5) {
    float *row = LT32 + m.lt_off + (size_t)k * m.n_pad;
    for (int j = threadIdx.x & 31; j < m.n_pad; j += 32)
      row[j] = (k < n && j < n && j >= k) ? (float)Li[(size_t)j * n + k] : 0.f;
  }
}

}  // namespace

constexpr int kMaxDevices = 64;

cudaError_t launch_fit(const SearchMeta *meta_d, int S, int smem_bytes, const FitIO &io,
                       SearchMeta *meta_out, cudaStream_t stream, bool pdl) {
  // the attribute call costs microseconds: only when it grows.  The attribute is per device, so
  // is the cache (one ctx per device may run in one process, on different threads)
  static std::atomic<int> smem_set[kMaxDevices];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices || smem_bytes > smem_set[dev].load()) {
    e = cudaFuncSetAttribute(fit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < kMaxDevices) {
      int cur = smem_set[dev].load();
      while (smem_bytes > cur && !smem_set[dev].compare_exchange_weak(cur, smem_bytes)) {
      }
    }
  }
  // programmatic dependent launch after the Gram pre-pass (see fit_body's griddepcontrol.wait);
  // the caller enables it for shared-memory working matrices only (n <= 216: fit 0.145 ->
  // 0.137 ms at n = 200; with the L2-resident matrix of n = 500 it measured 1.24 -> 1.34 ms)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(S);
  cfg.blockDim = dim3(kFitThreads);
  cfg.dynamicSmemBytes = (size_t)smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fit_kernel, meta_d, io, meta_out);
}

cudaError_t launch_gram(const SearchMeta *meta_d, int S, int nmax, int dmax, const FitIO &io,
                        cudaStream_t stream) {
  (void)dmax;
  const int nt = (nmax + 7) / 8;
  const int gx = std::max((nt * (nt + 1) / 2 + 3) / 4, (nmax + 127) / 128);
  gram_kernel<<<dim3(gx, S), 128, 0, stream>>>(meta_d, io);
  return cudaGetLastError();
}

cudaError_t launch_simt_operands(const SearchMeta *meta_d, int S, const float *X32,
                                 const float *ls32, const double *Linv64, float *Xs32,
                                 float *LT32, cudaStream_t stream) {
  simt_operands_kernel<<<S, 256, 0, stream>>>(meta_d, X32, ls32, Linv64, Xs32, LT32);
  return cudaGetLastError();
}

}  // namespace gpbo
