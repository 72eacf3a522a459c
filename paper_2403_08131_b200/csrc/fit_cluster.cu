// H2-H4 on a thread-block cluster: the fit of one sub-search spread over Cc CTAs (Cc <= 16, one
// cluster per search), float64 throughout.  PAPER.md L249/L256 (§IV.D): the GP's O(N^3) training.
//
// Same blocked elimination as fit.cu ([K | I] -> [L^T | L^-1] on 8 x 8 tiles, DMMA m8n8k4; the
// D / C / T phases of its header), but the working matrix W is DISTRIBUTED: CTA c owns the tile
// rows R = c (mod Cc) and keeps them in its own shared memory (row R's R + 1 tiles, row-major
// tiles, the DMMA fragment order).  Per 8-wide panel JT:
//   D  the owner of tile row JT factors the diagonal tile and forms the maps M, N, R (fit.cu),
//      then writes them and the pivot flag into every CTA of the cluster (DSMEM);
//   -- cluster barrier --
//   C  every CTA applies the maps to its own rows below the panel (the L panel and the panel's
//      row block of G); the owner of row JT also forms the final L^-1 block left of the panel;
//      each G value is stored into every CTA's copy of G (DSMEM);
//   -- cluster barrier --
//   T  every CTA runs the trailing update on its own rows with the full G; the owner of row JT + 1
//      first updates its diagonal tile and runs D(JT + 1) (look-ahead).
// The trailing update -- the O(n^3) bulk, shared-memory bound at ~25 cycles per tile and panel
// on one SM (fit.cu) -- is split Cc ways, and for n > 216 the matrix no longer lives
// in L2 (1 MB at n = 500 fits in 8 CTAs' shared memory).  Tail: each CTA writes its rows of L^-1
// (row-major), w_i = (L^-1 y~)_i and its partial alpha = L^-T w (column sums over its rows) to
// CTA 0, which adds the partials in rank order (deterministic) and writes alpha, the diagnostics
// and the meta record.  The jitter ladder restarts all CTAs together (the pivot flag travels
// with the maps).
#include <cooperative_groups.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>

#include "gpbo_internal.cuh"
#include "tc_prims.cuh"

namespace gpbo {
namespace {

namespace cg = cooperative_groups;
// 256 threads (255 registers) rather than the one-CTA fit's 384: config 4's 16-CTA fit
// 0.293 -> 0.266 ms measured (tools/ab_fit.sh); the one-CTA kernel is slower at 256 (0.108 -> 0.117)
#ifndef GPBO_FITC_THREADS
#define GPBO_FITC_THREADS 256
#endif
constexpr int kFitCThreads = GPBO_FITC_THREADS;
constexpr int kWarps = kFitCThreads / 32;
constexpr int kQ = 4;       // tiles of one tile row per trailing-update item
constexpr int kMaxCc = 16;  // 8 portable, 16 with the non-portable attribute

#ifdef GPBO_FIT_TIMING  // phase clocks of CTA (0, owner) printed at exit (tools/fit_phases.py)
#define FCT(slot) do { if (tid == 0) { const long long t_ = clock64(); ft[slot] += t_ - ft0; ft0 = t_; } } while (0)
#else
#define FCT(slot) do { } while (0)
#endif

// shared::cluster address of `saddr` (a shared::cta address) in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// bulk copy (TMA) local shared memory -> shared memory of another CTA of the cluster, completing
// `bytes` of transaction count on the destination CTA's mbarrier (both shared::cluster addresses)
__device__ __forceinline__ void bulk_s2s(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "r"(src), "r"(bytes), "r"(mbar) : "memory");
}

// bulk copy (TMA) global -> the same shared-memory offset in every CTA of `mask`, completing
// `bytes` of transaction count on each destination's mbarrier at the offset of `mbar`
__device__ __forceinline__ void bulk_g2s_mc(uint32_t dst, const void *src, uint32_t bytes,
                                            uint32_t mbar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1], %2, [%3], %4;"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar), "h"(mask) : "memory");
}

#ifndef GPBO_FITC_MCAST
#define GPBO_FITC_MCAST 1  // G rows via global staging + multicast (1) or DSMEM pushes (0)
#endif

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// 1 / sqrt(p) in float64: the float32 MUFU estimate (~2^-22, short latency; the float64 MUFU
// path is several times longer and sits on the D chain, this kernel's critical path) refined by
// two Newton steps (2^-44, then float64 rounding); p outside the float32 range takes the
// float64 estimate
__device__ __forceinline__ double rsqrt_fast(double p) {
  double y;
  if (p > 1e-30 && p < 1e30) {
    float yf;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"((float)p));
    y = (double)yf;
  } else {
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(p));
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double e = fma(-p, y * y, 1.0);
    y = fma(0.5 * y, e, y);
  }
  return y;
}

// tiles of the own rows R' = c, c + Cc, ... below R (R = c + lr Cc): sum_{i<lr} (c + i Cc + 1)
__host__ __device__ __forceinline__ int own_rowoff(int lr, int c, int Cc) {
  return lr * (c + 1) + Cc * lr * (lr - 1) / 2;
}

// shared-memory plan (doubles): yt | w | flags (24) | maps M N R (192) | L11 stash (64) |
// GT (2 x 8 nr8) | W (own tiles).  The GT area is reused by CTA 0 in the tail for the Cc partial
// alpha vectors (Cc x nr8 <= 16 nr8).
__host__ __device__ __forceinline__ int own_tiles(int nt, int c, int Cc) {
  const int rows = c < nt ? (nt - 1 - c) / Cc + 1 : 0;
  return own_rowoff(rows, c, Cc);
}

__global__ void __launch_bounds__(kFitCThreads, 1)
fit_cluster_kernel(const SearchMeta *__restrict__ meta_in, const FitIO io,
                   SearchMeta *__restrict__ meta_out) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[6 * kWarps + 8];
  cg::cluster_group cluster = cg::this_cluster();
  const int Cc = (int)cluster.num_blocks();
  const int c = (int)cluster.block_rank();
  const int s = blockIdx.x / Cc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  SearchMeta m = meta_in[s];
  if (io.sf2_src) { m.sf2 = io.sf2_src[s]; m.sn2 = io.sn2_src[s]; }
  const int n = m.n, d = m.d;
  const int nr8 = fit_nr8(n), gs = fit_gstride(n), nt = (n + 7) / 8;
  double *yt = sm;
  double *w = sm + nr8;
  double *flags = sm + 2 * nr8;   // [16]: pivot fail flag of the latest D
  double *Mm = flags + 24;
  double *Nm = Mm + 64;
  double *Rm = Nm + 64;
  double *l11s = Rm + 64;         // L11 of the latest D, written to global memory later
  // the panel's G transposed, double-buffered by panel parity: element (i, u) (row i of the
  // matrix, u = 0..7 the panel's columns) at gx(i, u) = 64 (i / 8) + 32 (u / 4) + 4 (i % 8) + u % 4:
  // a tile row is one contiguous 512-byte block (the unit of the DSMEM bulk copies) and a DMMA
  // fragment (rows gid, columns tig of one half) is 32 consecutive doubles -- conflict-free
  double *GT0 = l11s + 64;
  double *W = GT0 + 2 * 8 * nr8;
  auto gx = [](int i, int u) { return ((i >> 3) << 6) + ((u >> 2) << 5) + ((i & 7) << 2) + (u & 3); };
  double *G = GT0;  // (the tail reuses the GT area for CTA 0's partial alpha vectors)
  __shared__ __align__(8) uint64_t mbars[3];  // maps | G buffer 0 | G buffer 1
  // (DSMEM: every CTA's G, maps and flags sit at the same offsets; remote addresses are formed
  // with cluster.map_shared_rank where they are written)
  // Cc is a power of two (1, 2, 4, 8: api.cu fit_cluster_size): shifts instead of divisions
  const int lcc = __ffs(Cc) - 1;
  auto owner = [&](int R) { return R & (Cc - 1); };
  auto at = [&](int R, int C) -> double * {  // own tile (R, C), R = c (mod Cc)
    return W + (own_rowoff(R >> lcc, c, Cc) + C) * 64;
  };
  double *Lg = io.L64 + m.mat_off;
  const float *X = io.X_src + m.x_off;
  const float *ls = io.ls_src + m.ls_off;
  const double *y = io.y_src + m.y_off;

  // ---- validation (every CTA; CTA 0 copies the caller's device inputs into the model)
  const bool copy = io.X_src != io.X32 && c == 0;
  int bad = 0;
  for (int i = tid; i < n * d; i += kFitCThreads) bad |= !isfinite(X[i]);  // (X: copied by the pre-pass)
  for (int i = tid; i < n; i += kFitCThreads) {
    bad |= !isfinite(y[i]);
    if (copy) io.y64[m.y_off + i] = y[i];
  }
  for (int i = tid; i < d; i += kFitCThreads) {
    bad |= !(ls[i] > 0.f) || !isfinite(ls[i]);
    if (copy) io.ls32[m.ls_off + i] = ls[i];
  }
  bad |= !(m.sf2 > 0.f) || !isfinite(m.sf2) || !(m.sn2 >= 0.f) || !isfinite(m.sn2);
  bad = __syncthreads_or(bad);
  if (bad) {
    if (tid == 0 && c == 0) {
      m.status = GPBO_EINVAL; m.jitter_k = -1; m.lml = -INFINITY; meta_out[s] = m;
    }
    cluster.sync();
    return;
  }
  // ---- H1 (every CTA, identical arithmetic): y~ = (y - mean) / std, ddof 0 (R7 / R7a)
  auto bred = [&](double v, int op) {  // 0 sum, 1 max, 2 min; deterministic
    auto f = [op](double a, double b) { return op == 0 ? a + b : op == 1 ? fmax(a, b) : fmin(a, b); };
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = f(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = red[0];
    for (int i = 1; i < kWarps; ++i) t = f(t, red[i]);
    return t;
  };
  double acc = 0.0, amax = 0.0;
  for (int i = tid; i < n; i += kFitCThreads) { acc += y[i]; amax = fmax(amax, fabs(y[i])); }
  const double mean = bred(acc, 0) / n;
  amax = bred(amax, 1);
  acc = 0.0;
  for (int i = tid; i < n; i += kFitCThreads) { const double t = y[i] - mean; acc += t * t; }
  double stdv = sqrt(bred(acc, 0) / n);
  const bool degenerate = !(stdv > 1e-12 * amax);
  if (degenerate) stdv = 1.0;
  double bmin = INFINITY;
  for (int i = tid; i < n; i += kFitCThreads) {
    const double t = degenerate ? 0.0 : (y[i] - mean) / stdv;
    yt[i] = t;
    bmin = fmin(bmin, t);
  }
  const double best = bred(bmin, 2);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the Gram pre-pass is complete
  double pmax = 0.0;
  for (int b = 0; b * 128 < n; ++b) pmax = fmax(pmax, io.pm_part[16 * s + b]);
  const double sf2 = m.sf2, sn2 = m.sn2;

  // D (one warp of the owner of tile row J/8): as fit.cu's diag_block, then the maps and the
  // pivot flag go to every CTA of the cluster
  // D, warp-parallel: the elimination [A | I] -> [L^T | L^-1] of the 8 x 8 diagonal block (the
  // whole algorithm's step at 8 x 8 scale; E A = L^T with E = L^-1), lane l holding row l / 4,
  // columns 4 (l % 4) .. + 3 of the 8 x 16 array; per step one pivot and one row broadcast by
  // shuffles (the one-thread version of fit.cu took ~4-6 k cycles, on this kernel's critical
  // path).  Outputs: Nm = L11 (row-major lower, also stashed for the deferred global write),
  // Rm = X = L11^-1 (lower), flags[16] = a pivot <= 0 / non-finite.
  auto diag_block = [&](int J) {
    const int bb = min(kFitB, n - J);
    double *Wd = at(J >> 3, J >> 3);
    {
      const int i = lane >> 2, cb = 4 * (lane & 3);
      double v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = cb + e;
        if (col < 8)
          v[e] = (i < bb && col < bb) ? (col <= i ? Wd[8 * i + col] : Wd[8 * col + i])
                                      : (i == col ? 1.0 : 0.0);
        else
          v[e] = col - 8 == i ? 1.0 : 0.0;
      }
      bool fail = false;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double pj = __shfl_sync(0xffffffffu, v[j & 3], 4 * j + (j >> 2));
        fail |= !(pj > 0.0) || !isfinite(pj);
        const double r = rsqrt_fast(pj);
        const double bij = __shfl_sync(0xffffffffu, v[j & 3], 4 * i + (j >> 2));
        double rj[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) rj[e] = __shfl_sync(0xffffffffu, v[e], 4 * j + (lane & 3));
        if (i > j) {
          const double f = bij * r * r;  // B[i][j] / p
#pragma unroll
          for (int e = 0; e < 4; ++e) v[e] = fma(-f, rj[e], v[e]);
        } else if (i == j) {
#pragma unroll
          for (int e = 0; e < 4; ++e) v[e] *= r;
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = cb + e;
        if (col < 8) {
          if (col >= i) Nm[8 * col + i] = v[e];  // L11[col][i] = B[i][col]
        } else {
          Rm[8 * i + col - 8] = col - 8 <= i ? v[e] : 0.0;  // X[i][col - 8]
        }
      }
      if (lane == 0) flags[16] = fail ? 1.0 : 0.0;
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // L11 for the deferred global write (dl11 stash)
      const int e = lane + 32 * h, i = e >> 3, k = e & 7;
      l11s[e] = (k <= i && i < bb) ? Nm[e] : 0.0;
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
    double mv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h, mr = e >> 3, mc = e & 7;
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) t = fma(Rm[q * 8 + mr], Rm[q * 8 + mc], t);
      mv[h] = -t;
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) Mm[lane + 32 * h] = mv[h];
  };
  // the D warp of the owner: its maps block (flags | M | N | R, 1728 bytes) to every other CTA
  // by bulk copies (TMA) completing on their maps mbarrier, then its own arrival
  constexpr uint32_t kMapBytes = (24 + 192) * 8;
  const uint32_t mb_maps = tc::smem_u32(&mbars[0]);
  auto broadcast_maps = [&]() {
    tc::fence_proxy_async();  // the warp's generic writes -> visible to the async proxy
    __syncwarp();
    if (lane < Cc && lane != c)
      bulk_s2s(mapa(tc::smem_u32(flags), lane), tc::smem_u32(flags), kMapBytes,
               mapa(mb_maps, lane));
    if (lane == 0) tc::mbar_arrive(mb_maps);
  };

  // W(R, C0 + q) -= sum_u G[u][i] G[u][k], q < cnt (own row R), G = GT of the panel
  auto quad = [&](const double *GT, int R, int C0, int cnt) {
    const int i = 8 * R + gid;
    double *Wt = at(R, C0) + 2 * lane;
    double2 cc[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q)
      if (q < cnt) cc[q] = *reinterpret_cast<const double2 *>(Wt + 64 * q);
    (void)i;
    const double *ga = GT + R * 64 + gid * 4 + tig;
    const double a0 = -ga[0], a1 = -ga[32];
    const double *g = GT + C0 * 64 + gid * 4 + tig;
    double b0[kQ], b1[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q)
      if (q < cnt) { b0[q] = g[64 * q]; b1[q] = g[64 * q + 32]; }
#pragma unroll
    for (int q = 0; q < kQ; ++q)
      if (q < cnt) dmma(cc[q].x, cc[q].y, a0, b0[q]);
#pragma unroll
    for (int q = 0; q < kQ; ++q)
      if (q < cnt) dmma(cc[q].x, cc[q].y, a1, b1[q]);
#pragma unroll
    for (int q = 0; q < kQ; ++q)
      if (q < cnt) *reinterpret_cast<double2 *>(Wt + 64 * q) = cc[q];
  };

  // quad() for a full quad: no per-tile predicates (a predicated mma.sync costs a WARPSYNC + NOP
  // pair per DMMA), one base address per operand stream
  auto quad_full = [&](const double *__restrict__ GT, int R, int C0) {
    double *Wt = at(R, C0) + 2 * lane;
    double2 cc[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) cc[q] = *reinterpret_cast<const double2 *>(Wt + 64 * q);
    const double *ga = GT + R * 64 + gid * 4 + tig;
    const double a0 = -ga[0], a1 = -ga[32];
    const double *g = GT + C0 * 64 + gid * 4 + tig;
    double b0[kQ], b1[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) { b0[q] = g[64 * q]; b1[q] = g[64 * q + 32]; }
#pragma unroll
    for (int q = 0; q < kQ; ++q) dmma(cc[q].x, cc[q].y, a0, b0[q]);
#pragma unroll
    for (int q = 0; q < kQ; ++q) dmma(cc[q].x, cc[q].y, a1, b1[q]);
#pragma unroll
    for (int q = 0; q < kQ; ++q) *reinterpret_cast<double2 *>(Wt + 64 * q) = cc[q];
  };

  const int nown = c < nt ? (nt - 1 - c) / Cc + 1 : 0;  // own tile rows
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) tc::mbar_init(tc::smem_u32(&mbars[b]), 1);
    tc::fence_mbar_init();
  }
  cluster.sync();  // every CTA's mbarriers are initialised before any copy can target them
  uint32_t mp = 0, gp[2] = {0u, 0u};  // completed phases: maps barrier, G barriers
#ifdef GPBO_FIT_TIMING
  long long ft[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long wgs[3] = {0, 0, 0};
  long long ft0 = clock64();
  __shared__ long long dclk;
  if (tid == 0) dclk = 0;
#endif
  // every CTA waits for the maps of the current block: the owner arrived after its D, the others
  // arrive expecting the maps' bytes
  auto wait_maps = [&](int JT) {
    if (tid == 0 && owner(JT) != c) tc::mbar_arrive_expect_tx(mb_maps, kMapBytes);
    tc::mbar_wait(mb_maps, mp & 1u);
    ++mp;
  };
  int jk = -1;
  double jit = 0.0, p10 = 1.0;
  for (int k = 0; k < 7 && jk < 0; ++k, p10 *= 10.0) {
    jit = 1e-8 * p10 * sf2;
    // a restart of the ladder: every CTA has read the failing D's flag (and left the failed
    // sweep) before CTA 0's new maps(0) can overwrite its maps block
    if (k > 0) cluster.sync();
    __syncthreads();
    // H2: own rows' kernel tiles from the pre-pass, + sn2 + jitter on the diagonal
    for (int lr = 0; lr < nown; ++lr) {
      const int R = c + lr * Cc;
      const double2 *src = reinterpret_cast<const double2 *>(io.Kt64 + m.kt_off + (R * (R + 1) / 2) * 64);
      double2 *dst = reinterpret_cast<double2 *>(at(R, 0));
      for (int e = tid; e < (R + 1) * 32; e += kFitCThreads) dst[e] = src[e];
    }
    __syncthreads();
    for (int i = tid; i < n; i += kFitCThreads)
      if (owner(i >> 3) == c) at(i >> 3, i >> 3)[8 * (i & 7) + (i & 7)] += sn2 + jit;
    __syncthreads();
    FCT(0);
    if (c == 0 && warp == kWarps - 1) {
      diag_block(0);
      broadcast_maps();
    }
    __syncthreads();  // (the mbarrier already orders the maps; explicit for the race checker)
    FCT(1);
    wait_maps(0);
    FCT(2);
    bool ok = flags[16] == 0.0;
    for (int JT = 0; JT < nt && ok; ++JT) {
      const int J = 8 * JT, bb = min(kFitB, n - J);
      const int par = JT & 1;
      double *GT = GT0 + par * 8 * nr8;
      double *GS = io.G64 + m.stg_off + par * 8 * nr8;  // the same layout in global memory
      const int r0 = JT + 1 + ((c - (JT + 1)) & (Cc - 1));  // first own row > JT
      const int nrows = r0 < nt ? ((nt - 1 - r0) >> lcc) + 1 : 0;
      // ---- C: own rows below the panel; the owner of row JT also the block row left of it
      {
        const int nleft = owner(JT) == c ? JT : 0;
        for (int it = warp; it < nrows + nleft; it += kWarps) {
          double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
          if (it < nrows) {
            const int R = r0 + it * Cc, i = 8 * R + gid;
            double *Wt = at(R, JT);
#pragma unroll
            for (int kk = 0; kk < 8; kk += 4) {
              const double a = Wt[8 * gid + kk + tig];
              dmma(d0, d1, a, Nm[(kk + tig) * 8 + gid]);
              dmma(e0, e1, a, Mm[(kk + tig) * 8 + gid]);
            }
            // (the L panel goes to global memory in T); u = 2 tig, 2 tig + 1: one 16-byte store
            *reinterpret_cast<double2 *>(GT + gx(i, 2 * tig)) = make_double2(d0, d1);
            if (GPBO_FITC_MCAST) *reinterpret_cast<double2 *>(GS + gx(i, 2 * tig)) = make_double2(d0, d1);
            __syncwarp();  // every lane's tile reads precede the write-back (racecheck-clean)
            *reinterpret_cast<double2 *>(Wt + 2 * lane) = make_double2(e0, e1);
          } else {
            const int C = it - nrows;
            double *Wt = at(JT, C);
#pragma unroll
            for (int kk = 0; kk < 8; kk += 4) {
              const int mrow = kk + tig;
              const double b = mrow < bb ? Wt[8 * mrow + gid] : 0.0;
              dmma(d0, d1, Rm[gid * 8 + mrow], b);
            }
            const int kc = 8 * C + 2 * tig;
            GT[gx(kc, gid)] = d0;
            GT[gx(kc + 1, gid)] = d1;
            if (GPBO_FITC_MCAST) { GS[gx(kc, gid)] = d0; GS[gx(kc + 1, gid)] = d1; }
            __syncwarp();
            *reinterpret_cast<double2 *>(Wt + 2 * lane) = make_double2(d0, d1);
          }
        }
      }
      tc::fence_proxy_async();  // GT writes -> visible to the bulk copies below
      if (GPBO_FITC_MCAST) asm volatile("fence.proxy.async.global;" ::: "memory");  // GS too
      __syncthreads();
      FCT(3);
      if (JT + 1 == nt) {  // the last block: its L11 (no rows below, no trailing update)
        if (owner(JT) == c)
          for (int e = tid; e < 64; e += kFitCThreads) {
            const int i = e >> 3, k = e & 7;
            if (k <= i && i < bb) Lg[(size_t)(J + k) * n + J + i] = l11s[e];
          }
        break;
      }
      // ---- send this CTA's part of G (its rows below the block; the owner also the block row
      // left of it) to every other CTA: 512-byte tile-row blocks, warp 0 issuing
      const uint32_t mb_g = tc::smem_u32(&mbars[1 + par]);
      if (warp == 0 && GPBO_FITC_MCAST) {
        // one multicast bulk copy per own tile row (and the block row left of the panel at its
        // owner) from the global staging into every other CTA: the DSMEM pushes took 7 copies
        // per block, issued by one warp, and the owner's left block (up to 32 KB x 7) left its
        // SM serially; the multicast reads L2 once and fans out
        const uint16_t others = (uint16_t)(((1u << Cc) - 1u) & ~(1u << c));
        const int nl = owner(JT) == c && JT > 0 ? 1 : 0;
        for (int q = lane; q < nrows + nl; q += 32) {
          const uint32_t off = q < nrows ? (uint32_t)(r0 + q * Cc) * 512u : 0u;
          const uint32_t bytes = q < nrows ? 512u : 512u * (uint32_t)JT;
          if (others)
            bulk_g2s_mc(tc::smem_u32(GT) + off, reinterpret_cast<const char *>(GS) + off, bytes,
                        mb_g, others);
        }
      }
      if (warp == 0 && !GPBO_FITC_MCAST) {
        const int nl = owner(JT) == c && JT > 0 ? 1 : 0;
        const int items = (nrows + nl) * (Cc - 1);
        for (int it = lane; it < items; it += 32) {
          const int dst = it % (Cc - 1), q = it / (Cc - 1);
          const int r = dst < c ? dst : dst + 1;
          const uint32_t off = q < nrows ? (uint32_t)(r0 + q * Cc) * 512u : 0u;
          const uint32_t bytes = q < nrows ? 512u : 512u * (uint32_t)JT;
          const uint32_t src = tc::smem_u32(GT) + off;
          bulk_s2s(mapa(src, r), src, bytes, mapa(mb_g, r));
        }
      }
      if (warp == 0 && lane == 0) {  // this CTA's own arrival, expecting what the others send it:
        // the rows JT + 1 .. nt - 1 it does not own, and the left block unless it owns row JT
        const uint32_t expect = 512u * (uint32_t)(nt - 1 - JT - nrows) +
                                (owner(JT) != c ? 512u * (uint32_t)JT : 0u);
        tc::mbar_arrive_expect_tx(mb_g, expect);
      }
      // ---- deferred global writes of panel JT (their latency overlaps T): the L panel of the
      // own rows below the block (= their G entries) and, at the block's owner, the L11 of D(JT)
      for (int R = r0; R < nt; R += Cc)
        for (int e = tid; e < 64; e += kFitCThreads) {
          const int u = e >> 3, i = 8 * R + (e & 7);
          if (i < n) Lg[(size_t)(J + u) * n + i] = GT[gx(i, u)];
        }
      if (owner(JT) == c)
        for (int e = tid; e < 64; e += kFitCThreads) {
          const int i = e >> 3, k = e & 7;
          if (k <= i && i < bb) Lg[(size_t)(J + k) * n + J + i] = l11s[e];
        }
      __syncthreads();  // l11s and the maps are rewritten by the look-ahead D below
      // ---- T: own rows R > JT once every CTA's G has arrived; the owner of row JT + 1 first
      // updates its diagonal tile and runs D(JT + 1) (look-ahead; only its own G rows needed)
      {
        const bool look = owner(JT + 1) == c;
        const int nlq = (JT + kQ - 1) / kQ;
        const int kT = look ? kWarps - 1 : kWarps;
        if (look && warp == kWarps - 1) {
#ifdef GPBO_FIT_TIMING
          const long long td0 = clock64();
#endif
          quad(GT, JT + 1, JT + 1, 1);
          __syncwarp();
          diag_block(8 * (JT + 1));
          // every CTA has finished C(JT) (it sent its G) before its maps are overwritten
          tc::mbar_wait(mb_g, gp[par] & 1u);
          broadcast_maps();
#ifdef GPBO_FIT_TIMING
          if (lane == 0) dclk += clock64() - td0;
#endif
        } else {
#ifdef GPBO_FIT_TIMING
          const long long tw0 = clock64();
#endif
          tc::mbar_wait(mb_g, gp[par] & 1u);
#ifdef GPBO_FIT_TIMING
          if (tid == 0) wgs[(3 * JT) / nt] += clock64() - tw0;
#endif
          FCT(4);
          // items of own row R (r = R - JT - 1): nlq left quads (C < JT), then right quads of
          // columns JT + 1 .. R (row JT + 1's right quad is the diagonal tile: the D warp's)
          // (items are numbered row after row and dealt round robin: this warp's first item of
          // a row follows from the row's base number -- one modulo per row, not per item: the
          // per-item test was ~37 % of the kernel's instructions)
          int base = 0;
          for (int lr = 0; lr < nrows; ++lr) {
            const int R = r0 + lr * Cc, r = R - JT - 1;
            const int len = nlq + (r > 0 ? r / kQ + 1 : 0);
            const int q0 = (warp - base % kT + kT) % kT;
            base += len;
            for (int q = q0; q < len; q += kT) {
              int C0, cnt;
              if (q < nlq) {
                C0 = kQ * q;
                cnt = min(kQ, JT - kQ * q);
              } else {
                const int c0 = kQ * (q - nlq);
                C0 = JT + 1 + c0;
                cnt = min(kQ, r + 1 - c0);
              }
              if (cnt == kQ) quad_full(GT, R, C0);
              else quad(GT, R, C0, cnt);
            }
          }
        }
        ++gp[par];
      }
      __syncthreads();
      FCT(5);
      wait_maps(JT + 1);  // maps of D(JT + 1) and its pivot flag
      FCT(6);
      ok = flags[16] == 0.0;
    }
    if (ok) jk = k;
  }
  __syncthreads();
  if (jk < 0) {
    if (tid == 0 && c == 0) {
      m.status = GPBO_ENOTPD; m.jitter_k = -1; m.jitter = NAN; m.lml = -INFINITY;
      m.mean = mean; m.std = stdv; m.best = best; m.alpha_l1 = 0.0;
      meta_out[s] = m;
    }
    cluster.sync();
    return;
  }
  // ---- tail on own rows: row-major L^-1, w = L^-1 y~, row abs sums, abs max, log det, |w|^2
  double rs = 0.0, lam = 0.0, ld = 0.0, ww = 0.0;
  for (int lr = warp; lr < nown; lr += kWarps) {
    const int R = c + lr * Cc, i = 8 * R + gid;
    double a2 = 0.0, a3 = 0.0;
    double *dst = io.Linv64 + m.mat_off + (size_t)min(i, n - 1) * n;
    for (int C = 0; C <= R; ++C) {
      const double2 v = *reinterpret_cast<const double2 *>(at(R, C) + 2 * lane);
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
  // partial alpha_k = sum over own rows i >= k of (L^-1)_ik w_i, into CTA 0's slot c (DSMEM);
  // G is free now: CTA 0 keeps the Cc partial vectors there (Cc x nr8 <= 8 x gs doubles)
  double *part0 = cluster.map_shared_rank(G, 0) + (size_t)c * nr8;
  for (int C = warp; C < nt; C += kWarps) {
    const int c0 = 8 * C + 2 * tig;
    double s0 = 0.0, s1 = 0.0;
    const int rfirst = C + ((c - C % Cc) + Cc) % Cc;  // first own row >= C
    for (int R = rfirst; R < nt; R += Cc) {
      const int i = 8 * R + gid;
      if (i < n) {
        const double2 v = *reinterpret_cast<const double2 *>(at(R, C) + 2 * lane);
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
      if (c0 < nr8) part0[c0] = s0;
      if (c0 + 1 < nr8) part0[c0 + 1] = s1;
    }
  }
  // per-CTA statistics to CTA 0's flags area (slots 4 c .. 4 c + 3 of Mm, free after the sweep)
  {
    const double v0 = bred(rs, 1), v1 = bred(lam, 1), v2 = bred(ld, 0), v3 = bred(ww, 0);
    if (tid == 0) {
      double *st0 = cluster.map_shared_rank(Mm, 0) + 4 * c;
      st0[0] = v0; st0[1] = v1; st0[2] = v2; st0[3] = v3;
    }
  }
  cluster.sync();  // partials and statistics have landed in CTA 0
  FCT(7);
#ifdef GPBO_FIT_TIMING
  if (tid == 0 && s == 0 && (c == 0 || c == 1))
    printf("FITC n=%d Cc=%d c=%d load=%lld D0=%lld maps0=%lld C=%lld waitG=%lld T=%lld maps=%lld tail=%lld Dlook=%lld"
           " [G wait by panel third: %lld %lld %lld]\n",
           n, Cc, c, ft[0], ft[1], ft[2], ft[3], ft[4], ft[5], ft[6], ft[7], dclk, wgs[0], wgs[1], wgs[2]);
#endif
  if (c != 0) return;
  double l1 = 0.0, amx = 0.0;
  for (int k2 = tid; k2 < n; k2 += kFitCThreads) {
    double a = 0.0;
    for (int r = 0; r < Cc; ++r) a += G[(size_t)r * nr8 + k2];  // rank order: deterministic
    io.alpha64[m.a_off + k2] = a;
    l1 += fabs(a);
    amx = fmax(amx, fabs(a));
  }
  for (int kk = n + tid; kk < m.n_pad; kk += kFitCThreads) io.alpha64[m.a_off + kk] = 0.0;
  l1 = bred(l1, 0);
  amx = bred(amx, 1);
  if (tid == 0) {
    double rs_ = 0.0, lam_ = 0.0, ld_ = 0.0, ww_ = 0.0;
    for (int r = 0; r < Cc; ++r) {
      rs_ = fmax(rs_, Mm[4 * r]);
      lam_ = fmax(lam_, Mm[4 * r + 1]);
      ld_ += Mm[4 * r + 2];
      ww_ += Mm[4 * r + 3];
    }
    m.status = degenerate ? GPBO_WDEGENERATE : GPBO_OK;
    m.jitter_k = jk; m.jitter = jit;
    m.mean = mean; m.std = stdv; m.best = best; m.alpha_l1 = l1;
    m.pmax = (float)pmax; m.alpha_max = (float)amx; m.linv_rowsum = (float)rs_;
    m.linv_absmax = lam_;
    m.lml = -0.5 * ww_ - ld_ - 0.5 * n * 1.8378770664093454836;
    m.mean_tier = (double)m.sf2 * l1 > kMeanTierL1 ? 1 : 0;
    meta_out[s] = m;
  }
}

}  // namespace

// dynamic shared memory (bytes) of a search with n points on a cluster of Cc CTAs
int fit_cluster_smem(int n, int Cc) {
  const int nt = (n + 7) / 8;
  int tiles = 0;
  for (int c = 0; c < Cc; ++c) tiles = std::max(tiles, own_tiles(nt, c, Cc));
  return (2 * fit_nr8(n) + 24 + 4 * 64 + 2 * 8 * fit_nr8(n) + tiles * 64) * 8;
}

// the kernel's dynamic shared memory limit: the device's opt-in per-block maximum minus the
// kernel's static shared memory (queried once)
static int max_dyn_smem() {
  static const int v = [] {
    int dev = 0, optin = 227 * 1024;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, fit_cluster_kernel) != cudaSuccess) {
      cudaGetLastError();
      return optin - 4096;
    }
    return optin - (int)fa.sharedSizeBytes;
  }();
  return v;
}

// whether clusters of 16 CTAs with `smem_bytes` each can be resident on this device
bool fit_cluster16_ok(int smem_bytes) {
  // per device, the largest size already verified (the query costs a few driver calls per fit)
  static std::atomic<int> verified[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return false; }
  if (dev >= 0 && dev < 64 && smem_bytes <= verified[dev].load()) return true;
  if (cudaFuncSetAttribute(fit_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
          cudaSuccess ||
      cudaFuncSetAttribute(fit_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           max_dyn_smem()) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16);
  cfg.blockDim = dim3(kFitCThreads);
  cfg.dynamicSmemBytes = (size_t)smem_bytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 16;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, fit_cluster_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (nclusters > 0 && dev >= 0 && dev < 64) {
    int cur = verified[dev].load();
    while (smem_bytes > cur && !verified[dev].compare_exchange_weak(cur, smem_bytes)) {
    }
  }
  return nclusters > 0;
}

cudaError_t launch_fit_cluster(const SearchMeta *meta_d, int S, int Cc, int smem_bytes,
                               const FitIO &io, SearchMeta *meta_out, cudaStream_t stream) {
  // the attribute at the device maximum, once per device: never lowered below a size another
  // launch (or fit_cluster16_ok's query) relies on
  static std::atomic<int> smem_set[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (smem_bytes > max_dyn_smem()) return cudaErrorInvalidValue;
  if (dev < 0 || dev >= 64 || !smem_set[dev].load()) {
    e = cudaFuncSetAttribute(fit_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             max_dyn_smem());
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) smem_set[dev].store(1);
  }
  if (Cc > 8) {  // 16-CTA clusters are non-portable: opt in (once per device, like the smem)
    e = cudaFuncSetAttribute(fit_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(S * Cc);
  cfg.blockDim = dim3(kFitCThreads);
  cfg.dynamicSmemBytes = (size_t)smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = Cc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, fit_cluster_kernel, meta_d, io, meta_out);
}

}  // namespace gpbo
