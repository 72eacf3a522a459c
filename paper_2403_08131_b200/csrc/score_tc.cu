// Fast phase of H6-H9 on the 5th-generation tensor cores (tcgen05, TMEM, bulk-copy TMA).
//
// Per 128-candidate tile (M = 128, cta_group::1), per 32-wide panel p of training points:
//   (1) distance MMA  h = A_aug . B_aug^T into a TMEM scratch stage, with the augmented operands
//       A_aug = [x^*, |x^*|^2, 1], B_aug = [-2 x_j, 1, |x_j|^2] (x^ = x/l scaled so that h is
//       the kernel argument: 5 r^2 for Matern-5/2, r^2/2 for RBF) -- the "GEMM-form squared
//       distances on tensor cores" of the north star (a);
//   (2) epilogue warps: tcgen05.ld the scratch, K* = k(h) (MUFU sqrt/ex2 + FMA polynomial),
//       split K* into float16 hi + lo and store the panel as the A operand of (3);
//   (3) variance MMA  V[:, j >= 32p] += K*_p . (L^-1)[j, k in p]^T  into a TMEM accumulator of
//       n16 + 16 columns: the triangular "panel TRSM" V = L^-1 K*^T of north star (c), with L^-1
//       inverted at fit time; the k-step 16 of the panel only touches columns j >= 16 s.  The
//       16 extra B rows of every panel (score_pack.cuh, kMeanRows) make the same MMAs accumulate
//       mu~ = K* alpha and sum K* |alpha| (the mean error bound) in columns n16.. -- the mean of
//       north star (b) on the tensor cores, not on the epilogue's FMA pipe.
// After the last panel the epilogue drains V (sum V_j^2), forms s2~ = sf2 - |v|^2, EI and the
// EI bracket, and flags the candidates that can still be the argmax for the float64 refine
// phase (refine.cu) -- north star (d).
//
// Precision: every operand is split x = hi + lo in float16 (hi = x truncated to 11 bits, lo the
// exact remainder rounded to float16) and each contraction issues hi.hi + hi.lo + lo.hi, giving
// float32-level (22-bit) products with float32 accumulation; power-of-two scales (pack_tc) keep
// the float16 operands in range.  1x float16/bf16/tf32 would break the 1e-4 parity
// (SURVEY.md Appendix A).
//
// Warp roles (512 threads, one persistent CTA per SM, static contiguous tile ranges):
//   warps 0-7   K* (2 warps per TMEM lane quarter, 32 training points of each panel each)
//   warps 8-11  drain + finish of the previous tile (overlaps the K* work of the next one)
//   warps 12-13 candidate loader (X* -> A_aug)
//   warp 14     TMEM allocator, image TMA, distance MMA issuer
//   warp 15     variance MMA issuer (warp-uniform, one elected lane issues)
// The issue arbiter of an SM sub-partition favours the highest warp id (B300_MICROARCH.md), so
// the latency-critical MMA issuer gets the highest id and is never starved by the epilogue.
// Shared memory: the per-search operand image (X^ rows, L^-1 panels, alpha, candidate scales)
// is loaded once per search segment with one bulk copy and stays resident; the candidate tile
// and two K* panel stages are the only per-tile operands.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "score_common.cuh"
#include "score_tc.cuh"
#include "tc_prims.cuh"
#include "score_tc_helpers.cuh"
#include "score_pack.cuh"

namespace gpbo {

namespace {

// K* warps: 2 per sub-partition (8), each evaluating 32 of a panel's 64 training points;
// -DGPBO_KWARPS=16 builds 4 per sub-partition x 16 points (measured: config 2 fast phase
// 0.254 -> 0.275 ms -- the K* warps then wait on the MMA handoffs instead, and the 768-thread
// block caps registers at 80; config 3 -2 %).
#ifndef GPBO_KWARPS
#define GPBO_KWARPS 8
#endif
constexpr int kKWarps = GPBO_KWARPS;
static_assert(kKWarps == 8 || kKWarps == 16, "K* warps: 2 or 4 per TMEM lane quarter");
constexpr int kCW = 256 / kKWarps;           // training points per K* warp and panel (32 / 16)
constexpr int kDrainW0 = kKWarps;            // drain + finish warps kDrainW0 .. + 3
constexpr int kLoadW0 = kKWarps + 4;         // candidate loader warps kLoadW0, + 1
constexpr int kDistW = kKWarps + 6;          // TMEM allocator, image TMA, distance MMA issuer
constexpr int kVarW = kKWarps + 7;           // variance MMA issuer (highest warp id)
constexpr int kThreads = 32 * (kKWarps + 8);
constexpr uint32_t kTmemCols = 512;
constexpr int kMaxSmem = 227 * 1024;
constexpr int kStageBytes = 16384;  // one K* panel stage: hi (128 x 64 B) + lo (128 x 64 B)
constexpr int kDepth = 2;           // 64-column distance scratch stages (TMEM), issued ahead
constexpr int kKStages = 2;         // K* operand stages (TMEM), one 64-wide panel each
// TMEM columns: V accumulator [0, n16 + 16 <= 256), distance scratch 2 x 64 [256, 384), K* operand
// stages 2 x 64 [384, 512) (per stage: hi k-steps 0..3 at +0/+8/+16/+24, lo at +32..+56;
// lane = row, one column packs the fp16 pair k = 2c, 2c+1).  A K* panel is 64 training points
// wide (= one distance chunk): every TMEM round trip of the K* warps (distance load, K* store,
// their waits and barrier handoffs) is paid once per 64 points -- those latencies, not the
// MUFU or tensor pipes, bound the kernel (timing experiments without MUFU work / without 2/3
// of the MMAs: -7 % / -4 %).
constexpr uint32_t kScratch0 = 256;
// GPBO_RING4: kMerged launches (every n16 + 16 <= 128) trade the second V accumulator for a
// 4-deep distance ring: V [0, 128), ring [128, 384), K* stages [384, 512)
#ifndef GPBO_RING4
#define GPBO_RING4 1  // measured: config 3 fast phase 2.689 -> 2.653 ms (config 2: not kMerged, unaffected)
#endif
constexpr uint32_t kKstar0 = 384;

enum {
  B_AF0 = 0, B_AF1, B_AE0, B_AE1,           // candidate A tile (double buffer)
  B_DF0, B_DF1, B_DF2, B_DF3, B_DE0, B_DE1, B_DE2, B_DE3,  // distance scratch ring (<= 4)
  B_KF0, B_KF1, B_KF2, B_KF3, B_KE0, B_KE1, B_KE2, B_KE3,  // K* panel stages
  B_VF0, B_VF1, B_VE0, B_VE1,               // V accumulators
  B_SF0, B_SF1,                             // raw candidate rows landed in staging (TMA)
  B_VB0, B_VB1, B_VB2, B_VB3,               // V column block [64 p, 64 p + 64) final (per panel)
  B_IMG, B_COUNT
};

enum : uint32_t { kFlagInvalid = 1u, kFlagUnsafe = 2u };

// dynamic shared memory: image | A tiles x2 | staging x2 | row info x8
struct TcSmem {
  int img, a, k, stage, rowinfo, bars, total;
};

__host__ __device__ inline TcSmem tc_smem(int img_max, int kb_max, int d_max) {
  TcSmem s;
  s.img = 0;
  s.a = img_max;
  s.k = s.a + 2 * kb_max * 8192;
  s.stage = s.k;
  s.rowinfo = s.stage + 2 * ((128 * d_max * 4 + 127) & ~127);
  s.bars = s.rowinfo + 8 * 128 * 8;
  s.total = s.bars + B_COUNT * 8 + 16 + 1024;  // + tmem slot, + alignment slack
  return s;
}

// kPair: a cluster of two CTAs on one TPC scores 256-candidate pair tiles with M = 256 MMAs
// (cta_group::2): each CTA holds its 128 rows (candidate tile, distances, K* stages, V) and half
// of every B operand (the search's half image, score_pack.cuh); CTA 0 issues every MMA for both,
// and every handoff, MMA issue and commit is paid once per 256 candidates.  The pair tile u of a
// search covers its 128-row tiles 2u (CTA 0) and 2u + 1 (CTA 1); the host gives every search an
// even tile count.
template <bool kMerged, bool kPair>
__global__ void __launch_bounds__(kThreads, 1)
score_tc_kernel(const ScoreLaunch p, int tile_lo, int total_tiles, int img_max, int kb_max, int d_max) {
  constexpr int kDep = (kMerged && GPBO_RING4) ? 4 : kDepth;                 // distance ring depth
  constexpr uint32_t kScr = (kMerged && GPBO_RING4) ? 128u : kScratch0;     // its first column
  extern __shared__ unsigned char sm_raw[];
  unsigned char *sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
  const TcSmem L = tc_smem(img_max, kb_max, d_max);
  unsigned char *img = sm + L.img;
  unsigned char *Abuf = sm + L.a;
  float *stage = reinterpret_cast<float *>(sm + L.stage);
  float2 *rowinfo = reinterpret_cast<float2 *>(sm + L.rowinfo);
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + L.bars);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + B_COUNT);
  auto bar = [&](int i) { return tc::smem_u32(bars + i); };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? tc::cluster_rank() : 0u;  // CTA of the pair (0 issues the MMAs)
  const bool leader = rank == 0u;
  constexpr int kTs = kPair ? 2 : 1;  // 128-row tiles per (pair) tile
  // this launch covers tiles [tile_lo, tile_lo + total_tiles) of the call (chunked host feeds);
  // ta / tb below count (pair) tiles: units of kTs 128-row tiles
  const int units = total_tiles / kTs, unit_lo = tile_lo / kTs;
  const int gid = kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int ngrp = kPair ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int t0 = unit_lo + (int)((long long)units * gid / ngrp);
  const int t1 = unit_lo + (int)((long long)units * (gid + 1) / ngrp);
  // an arrival on the issuing CTA's copy of a barrier (the pair's consumers of CTA 0's MMAs):
  // relaxed -- the arriving threads' TMEM loads / stores have completed (tcgen05.wait::ld/st)
  auto arrive_leader = [&](uint32_t b) {
    if (kPair) tc::mbar_arrive_cluster_relaxed(tc::mapa(b, 0u));
    else tc::mbar_arrive(b);
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      // (pair: one arrival per CTA's loader on CTA 0's barrier; else every loader thread)
      tc::mbar_init(bar(B_AF0 + i), kPair ? 2 : 64);
      tc::mbar_init(bar(B_AE0 + i), 1);

      tc::mbar_init(bar(B_VF0 + i), 1);
      tc::mbar_init(bar(B_VE0 + i), 4 * kTs);
      tc::mbar_init(bar(B_SF0 + i), 1);
    }
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(bar(B_DF0 + i), 1);
      tc::mbar_init(bar(B_DE0 + i), kKWarps * kTs);
    }
    for (int i = 0; i < kKStages; ++i) {
      tc::mbar_init(bar(B_KF0 + i), kKWarps * kTs);
      tc::mbar_init(bar(B_KE0 + i), 1);
    }
    for (int i = 0; i < 4; ++i) tc::mbar_init(bar(B_VB0 + i), 1);
    tc::mbar_init(bar(B_IMG), 1);
    tc::fence_mbar_init();
  }
  if (warp == kDistW) {
    if (kPair) tc::tmem_alloc2(tc::smem_u32(tmem_slot), kTmemCols);
    else tc::tmem_alloc(tc::smem_u32(tmem_slot), kTmemCols);
  }
  tc::tc_fence_before();
  if (kPair) tc::cluster_sync();  // both CTAs' barriers initialised before any remote arrival
  else __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  // programmatic dependent launch: barrier init and TMEM allocation above overlapped the
  // previous kernel (the operand pack); its outputs (meta constants, image) are read below.
  // The refine kernel may be scheduled on SMs this grid frees.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
#if defined(GPBO_TC_TRACE) || defined(GPBO_TC_CTATIME)
  unsigned long long cta_t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(cta_t0));
#endif

  // Counters are CTA-global across segments (mbarrier phases continue): tiles gi, distance
  // panels gd, K* panels gk.  Every role advances them identically.
  uint32_t gi = 0, gc_seg = 0, gk_seg = 0;
  uint32_t trc = 0;  // trace event count of this thread
  uint32_t img_phase = 0;
  // completions of B_VE0 / B_VE1 (V buffer freed) and of the block-barrier groups B_VB0..1 /
  // B_VB4..7 so far: the single- and double-buffered modes can alternate between segments
  uint32_t ve0 = 0, ve1 = 0, vb0c = 0, vb1c = 0;

  for (int ta = t0; ta < t1;) {
    // ---------------- segment [ta, tb): consecutive (pair) tiles of one search
    const int s = search_of(p.tile_first, p.S, kTs * ta);
    const int tb = min(t1, p.tile_first[s + 1] / kTs);
    const SearchMeta &m = p.meta[s];
    // previous segment fully drained (epilogue consumed the last commit; for the pair that
    // commit followed every MMA reading this CTA's half image, so it may be replaced)
    __syncthreads();
    if (threadIdx.x == 32 * kDistW) {
      tc::mbar_arrive_expect_tx(bar(B_IMG), (uint32_t)m.img_bytes);
      tc::bulk_g2s(tc::smem_u32(img), p.img + m.img_off + (int64_t)rank * m.img_bytes,
                   (uint32_t)m.img_bytes, bar(B_IMG));
    }
    tc::mbar_wait(bar(B_IMG), img_phase);
    img_phase ^= 1u;
    const int n16 = m.n16, npan = m.npan, kb = m.kb;
    // n16 + 16 <= 128: two V accumulators [0, 128) and [128, 256) alternate between tiles, so
    // the next tile's variance MMAs never wait for the previous tile's drain; block barriers
    // B_VB0..1 / B_VB2..3 per buffer.  Otherwise one accumulator and 4 block barriers (one per
    // 64-wide column block: one commit per panel besides the K* stage release).
    const int nv16 = n16 + kMeanRows;  // V accumulator columns (L^-1 rows + mean rows)
    const bool dbl = nv16 <= 128 && !(kMerged && GPBO_RING4);
    const uint32_t vbq = dbl ? 2u : 4u;
    const int T = tb - ta;
    const int P64 = (n16 + 63) / 64;  // 64-wide K* panels per tile
    const int P = T * P64;
    const int64_t Ms = p.m_off[s + 1] - p.m_off[s];
    // local 128-row tile index of this CTA's first tile of the segment (tile tl: tile0 + kTs tl)
    const int tile0 = kTs * ta + (int)rank - p.tile_first[s];

    if (warp == kDistW || warp == kVarW) {
      // the pair's second CTA issues nothing: its operands are read by CTA 0's MMAs
      if (!leader) {
      } else if (warp == kDistW) {
      // ===================================================== distance MMA issuer
      // 64-wide chunks (one chunk feeds two K* panels; a tcgen05.mma costs max(40, N/2)
      // cycles, so N = 64 halves the issue cost of N = 32), issued as soon as a TMEM ring stage
      // is free -- independent of the variance MMAs, so the K* warps never wait on them.
      const uint32_t H32 = tc::sdesc_hi(32);
      const uint32_t x0 = tc::sdesc_lo(tc::smem_u32(img));
      const uint32_t abase = tc::sdesc_lo(tc::smem_u32(Abuf));
      const uint32_t xlo = (uint32_t)(n16 * 32) >> 4;  // hi -> lo block of the X^ operand
      const int ndc = (npan + 1) >> 1;                 // distance chunks per tile
      uint32_t gc = gc_seg;
      int d_st = (int)(gc % kDep);
      uint32_t d_ph = (gc / kDep) & 1u;
      for (int tl = 0; tl < T; ++tl) {
        const uint32_t ti = gi + tl, ab = ti & 1u;
        tc::mbar_wait(bar(B_AF0 + ab), (ti >> 1) & 1u);
        tc::tc_fence_after();
        for (int q = 0; q < ndc; ++q) {
          tc::mbar_wait(bar(B_DE0 + d_st), d_ph ^ 1u);
          tc::tc_fence_after();
          const uint32_t Nq = (uint32_t)min(64, n16 - 64 * q);
          const uint32_t dt = tbase + kScr + 64u * (uint32_t)d_st;
          uint32_t a = abase + ab * (uint32_t)kb * 512u;  // 8192 B per K block
          if (lane == 0) trace_ev(p.trace, 24, 11, gc, trc);
          if constexpr (kPair) {
            // this CTA's half of chunk q: K block k hi at +2048 k, lo at +1024 (score_pack.cuh)
            const uint32_t idn = tc::idesc_f16_m256(Nq);
            uint32_t bq = x0 + (uint32_t)(q * kb) * 128u;
            for (int k = 0; k < kb; ++k) {
              tc::mma2_f16_split(dt, a, H32, bq, H32, idn, k > 0);
              tc::mma2_f16_split(dt, a, H32, bq + 64u, H32, idn, 1u);
              tc::mma2_f16_split(dt, a + 256u, H32, bq, H32, idn, 1u);  // A lo: +4096 B
              a += 512u;
              bq += 128u;
            }
            tc::mma2_commit_warp(bar(B_DF0 + d_st));
          } else {
            const uint32_t idn = tc::idesc_f16(Nq);
            uint32_t bq = x0 + (uint32_t)q * 128u;          // rows 64 q (2048 B)
            for (int k = 0; k < kb; ++k) {
              tc::mma_f16_split(dt, a, H32, bq, H32, idn, k > 0);
#ifndef GPBO_EXP_NODIST  // timing experiment only: 1 of the 3 distance products
              tc::mma_f16_split(dt, a, H32, bq + xlo, H32, idn, 1u);
              tc::mma_f16_split(dt, a + 256u, H32, bq, H32, idn, 1u);  // A lo: +4096 B
#endif
              a += 512u;
              bq += 2u * xlo;
            }
            tc::mma_commit_warp(bar(B_DF0 + d_st));
          }
          if (lane == 0) trace_ev(p.trace, 4, 11, gc, trc);
          ++gc;
          if (++d_st == kDep) { d_st = 0; d_ph ^= 1u; }
        }
        if (kPair) tc::mma2_commit_warp(bar(B_AE0 + ab));  // A tiles of both CTAs consumed
        else tc::mma_commit_warp(bar(B_AE0 + ab));         // A tile consumed
      }
      __syncwarp();
      } else {
      // ===================================================== variance MMA issuer
      {
        const uint32_t H64 = tc::sdesc_hi(64), H32v = tc::sdesc_hi(32);
        const uint32_t l0 = tc::sdesc_lo(tc::smem_u32(img + m.off_l));
        uint32_t gk = gk_seg;
        int v_tl = 0, v_pp = 0;
        for (int g = 0; g < P; ++g) {
          const uint32_t ks = gk % kKStages;
          if (lane == 0) trace_ev(p.trace, 1, 11, gk, trc);
          tc::mbar_wait(bar(B_KF0 + ks), (gk / kKStages) & 1u);
          if (lane == 0) trace_ev(p.trace, 2, 11, gk, trc);
          tc::tc_fence_after();
          const uint32_t vti = gi + (uint32_t)v_tl;
          const uint32_t vb = dbl ? (vti & 1u) : 0u;  // V buffer of this tile
          if (v_pp == 0) {
            tc::mbar_wait(bar(B_VE0 + vb), ((vb ? ve1 : ve0) & 1u) ^ 1u);
            tc::tc_fence_after();
          }
          const uint32_t kt = tbase + kKstar0 + 64u * ks;  // K* stage in TMEM
#pragma unroll
          for (int sk = 0; sk < 4; ++sk) {  // 16-wide k steps of the 64-wide panel
            const int j0 = 64 * v_pp + 16 * sk;
            if (j0 < n16) {
              const uint32_t dt = tbase + 128u * vb + (uint32_t)j0;
              const uint32_t ka = kt + 8u * sk;       // k step sk: hi at +8 sk, lo at +32 + 8 sk
              if constexpr (kPair) {
                // k-step slab j0 / 16 of this CTA's half image: hi (N / 2 rows x 32 B), then lo
                const uint32_t Nv = (uint32_t)(nv16 - j0);
                const uint32_t lb = l0 + ((uint32_t)tc_pair_slab(nv16, j0 >> 4) >> 4);
                const uint32_t idn = tc::idesc_f16_m256(Nv);
                tc::mma2_f16_ts(dt, ka, lb, H32v, idn, (v_pp | sk) ? 1u : 0u);
                tc::mma2_f16_ts(dt, ka, lb + Nv, H32v, idn, 1u);
                tc::mma2_f16_ts(dt, ka + 32u, lb, H32v, idn, 1u);
              } else {
                const int pp = 2 * v_pp + (sk >> 1), h = sk & 1;  // 32-wide L^-1 panel, k step
                const uint32_t R16 = (uint32_t)(nv16 - 32 * pp) * 4u;  // R * 64 B >> 4: hi -> lo
                const uint32_t lp = l0 + (uint32_t)(pp * nv16 - 16 * pp * (pp - 1)) * 8u;
                const uint32_t idn = tc::idesc_f16((uint32_t)(nv16 - j0));
                const uint32_t lb = lp + 66u * h;       // +1024 B rows, +32 B k-advance
                tc::mma_f16_ts(dt, ka, lb, H64, idn, (v_pp | sk) ? 1u : 0u);
#ifndef GPBO_EXP_NOVMMA
                tc::mma_f16_ts(dt, ka, lb + R16, H64, idn, 1u);
                tc::mma_f16_ts(dt, ka + 32u, lb, H64, idn, 1u);
#endif
              }
              if (lane == 0) trace_ev(p.trace, 20 + sk, 11, gk, trc);
            }
          }
          // the K* stage is free; V columns [64 q, 64 q + 64) receive no later contribution (the
          // drain may read them)
          if (kPair) {
            tc::mma2_commit_warp(bar(B_KE0 + ks));
            tc::mma2_commit_warp(bar(B_VB0 + vbq * vb + v_pp));
          } else {
            tc::mma_commit_warp(bar(B_KE0 + ks));
            tc::mma_commit_warp(bar(B_VB0 + vbq * vb + v_pp));
          }
          if (lane == 0) trace_ev(p.trace, 3, 11, gk, trc);
          ++gk;
          if (++v_pp == P64) {
            // the unused block barriers complete too: every B_VB completes once per tile
            for (int q = P64; q < (int)vbq; ++q) {
              if (kPair) tc::mma2_commit_warp(bar(B_VB0 + vbq * vb + q));
              else tc::mma_commit_warp(bar(B_VB0 + vbq * vb + q));
            }
            v_pp = 0;
            ++v_tl;
            if (vb) ++ve1; else ++ve0;
          }
        }
      }
      __syncwarp();
      }
    } else if (warp == kLoadW0 || warp == kLoadW0 + 1) {
      // ===================================================== candidate loader
      // Raw rows of tile t+1 are prefetched into the other staging buffer by one bulk copy
      // (TMA) while tile t is converted into the float16 hi/lo A operand.
      const int lt = threadIdx.x - 32 * kLoadW0;
      const int d = m.d;
      const float *w = reinterpret_cast<const float *>(img + m.off_w);
      const int stage_floats = ((128 * d_max * 4 + 127) & ~127) / 4;
      auto fetch = [&](int tl) {  // all 64 loader threads call it
        const uint32_t ti = gi + tl, sb = ti & 1u;
        const int64_t row0 = (int64_t)(tile0 + kTs * tl) * 128;
        // (a pair tile's second half may lie past the search's rows: nothing to copy)
        const int rows = (int)(Ms - row0 < 128 ? (Ms - row0 > 0 ? Ms - row0 : 0) : 128);
        const float *src = p.Xstar + p.x_off[s] + (rows > 0 ? row0 * d : 0);
        float *dst = stage + sb * stage_floats;
        const uint32_t bytes = (uint32_t)(rows * d * 4);
        if (rows > 0 && (((uintptr_t)src) & 15u) == 0 && (bytes & 15u) == 0) {
          if (lt == 0) {
            tc::mbar_arrive_expect_tx(bar(B_SF0 + sb), bytes);
            tc::bulk_g2s(tc::smem_u32(dst), src, bytes, bar(B_SF0 + sb));
          }
        } else {  // unaligned shard: plain loads, then a plain arrive completes the phase
          for (int e = lt; e < rows * d; e += 64) dst[e] = __ldg(src + e);
          tc::named_bar_sync(3, 64);
          if (lt == 0) tc::mbar_arrive(bar(B_SF0 + sb));
        }
      };
      if (T > 0) fetch(0);
      for (int tl = 0; tl < T; ++tl) {
        const uint32_t ti = gi + tl, ab = ti & 1u, sb = ti & 1u;
        const int64_t row0 = (int64_t)(tile0 + kTs * tl) * 128;
        if (tl + 1 < T) fetch(tl + 1);
        if (lt == 0) trace_ev(p.trace, 9, 8, ti, trc);
        tc::mbar_wait(bar(B_SF0 + sb), (ti >> 1) & 1u);
        tc::mbar_wait(bar(B_AE0 + ab), ((ti >> 1) & 1u) ^ 1u);
        if (lt == 0) trace_ev(p.trace, 10, 8, ti, trc);
        const int rows = (int)(Ms - row0 < 128 ? Ms - row0 : 128);  // (<= 0: all rows invalid)
        const float *stg = stage + sb * stage_floats;
        const uint32_t a0 = tc::smem_u32(Abuf) + ab * kb * 8192;
        for (int r = lt; r < 128; r += 64) {
          const bool valid = r < rows;
#ifndef GPBO_LOADER_SCALAR  // (A/B switch)
          if ((d & 3) == 0) {  // vectorised path (configs 2, 4)
            float qh;
            bool nan;
            convert_row_vec4(stg, w, r, d, kb, valid, a0, qh, nan);
            const bool unsafe = !(qh <= 30000.f);
            const uint32_t flags =
                (valid && !nan ? 0u : kFlagInvalid) | (unsafe ? kFlagUnsafe : 0u);
            rowinfo[(ti & 7u) * 128 + r] = make_float2(qh * m.hscale, __uint_as_float(flags));
            continue;
          }
#endif
          float qh = 0.f;
          bool nan = false;
          if (valid)
            for (int c = 0; c < d; ++c) {
              const float x = stg[r * d + c];
              nan |= !isfinite(x);
              const float v = x * w[c];
              qh = fmaf(v, v, qh);
            }
          const bool unsafe = !(qh <= 30000.f);
          for (int k = 0; k < kb; ++k) {
            uint32_t hw[8], lw[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float v2[2];
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const int c = 16 * k + 2 * q + u;
                float v = 0.f;
                if (valid && !unsafe) {
                  if (c < d) v = stg[r * d + c] * w[c];
                  else if (c == d) v = qh;
                  else if (c == d + 1) v = 1.f;
                }
                v2[u] = v;
              }
              const __half2 h2 = __floats2half2_rn(v2[0], v2[1]);
              const float2 hf = __half22float2(h2);
              hw[q] = *reinterpret_cast<const uint32_t *>(&h2);
              lw[q] = tc::pack_f16x2(v2[0] - hf.x, v2[1] - hf.y);
            }
            const uint32_t base = a0 + k * 8192;
            sts128(base + tc::sw_offset(r, 0, 32), hw[0], hw[1], hw[2], hw[3]);
            sts128(base + tc::sw_offset(r, 16, 32), hw[4], hw[5], hw[6], hw[7]);
            sts128(base + 4096 + tc::sw_offset(r, 0, 32), lw[0], lw[1], lw[2], lw[3]);
            sts128(base + 4096 + tc::sw_offset(r, 16, 32), lw[4], lw[5], lw[6], lw[7]);
          }
          const uint32_t flags =
              (valid && !nan ? 0u : kFlagInvalid) | (unsafe ? kFlagUnsafe : 0u);
          rowinfo[(ti & 7u) * 128 + r] = make_float2(qh * m.hscale, __uint_as_float(flags));
        }
        tc::fence_proxy_async();
        tc::named_bar_sync(3, 64);  // staging buffer sb free, A tile complete
        if (kPair) {  // one arrival per CTA on the issuing CTA's barrier (release: the A tile's
                      // shared-memory stores precede the MMA's reads)
          if (lt == 0) tc::mbar_arrive_cluster(tc::mapa(bar(B_AF0 + ab), 0u));
        } else {
          tc::mbar_arrive(bar(B_AF0 + ab));
        }
        if (lt == 0) trace_ev(p.trace, 11, 8, ti, trc);
      }
    } else if (warp >= kDrainW0 && warp < kDrainW0 + 4) {
      // ===================================================== drain + finish (4 warps)
      // One thread per candidate row: waits for the tile's V accumulator, sums V_j^2 over all
      // n16 columns, frees V, adds the K* warps' partial means, and finishes the tile (EI
      // bracket, threshold, refine list) -- while the K* warps already work on the next tile.
      const int lq = warp & 3;
      const int row = 32 * lq + lane;
      const uint32_t va0 = tbase + ((uint32_t)(32 * lq) << 16);
      const FinishSeg fs = finish_seg(p, s);  // per-search values, once per segment
      const int64_t row0s = p.m_off[s];
      const float vun2 = m.vunscale2, sf2 = m.sf2, pmaxh = m.pmax_h, lrs = m.linv_rowsum;
      const float mun = m.munscale;
      // absolute floor of the MMA mean's error: K* entries below the float16 range of the lo
      // part (|K*| 2^tK < 2^-14) are represented to 2^-25 2^-tK = 2^-38 sf2 (2^tK >= 2^12 / sf2),
      // so |d mu~| <= 2^-38 sf2 |alpha|_1; 4x margin
      const float dmu_abs = (float)((double)m.sf2 * m.alpha_l1 * 1.4551915228366852e-11);
      const int nn = m.n;
      const bool mtier = p.mean64 != nullptr && m.mean_tier;  // precise-mean tier (mean64.cu)
      // variance bound 4 var_bound(u, sf2, s2, n, lrs) = vbk (sf2 + s2), its factor hoisted
      const float vbk = 4.f * 16.f * 5.9604645e-8f * sqrtf((float)nn) * (1.f + 0.01f * lrs * sqrtf(sf2));
      for (int tl = 0; tl < T; ++tl) {
        const uint32_t ti = gi + tl;
        const uint32_t vb = dbl ? (ti & 1u) : 0u;
        const uint32_t va = va0 + 128u * vb;
        // progressive drain: column block p of V is final once panel p's MMAs complete (each
        // barrier of the buffer's block group completes once per tile on that buffer, and the
        // buffer's next tile cannot start before B_VE)
        const bool trd = warp == kDrainW0 && lane == 0;
        // the threshold read is issued before the V drain so its latency is hidden
        const float thr = p.mode == kModeArgmax ? read_thr(p, s) : 0.f;
        if (trd) trace_ev(p.trace, 16, 9, ti, trc);
        float vv = 0.f;
        for (int pb = 0; pb < npan; ++pb) {
          if ((pb & 1) == 0) {  // one barrier per 64-wide block (two 32-wide drain blocks)
            const uint32_t blk = vbq * vb + (uint32_t)(pb >> 1);
            tc::mbar_wait(bar(B_VB0 + blk), (vb ? vb1c : vb0c) & 1u);
            tc::tc_fence_after();
          }
          const int c = 32 * pb;
#ifdef GPBO_EXP_NODRAINLD  // timing experiment only: the drain does not read V
          if (false) {
#else
          if (c + 32 <= n16) {
#endif
            uint32_t r0[16], r1[16];
            tc::tmem_ld16(va + (uint32_t)c, r0);
            tc::tmem_ld16(va + (uint32_t)(c + 16), r1);
            tc::tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const float v0 = __uint_as_float(r0[q]), v1 = __uint_as_float(r1[q]);
              vv = fmaf(v0, v0, vv);
              vv = fmaf(v1, v1, vv);
            }
          } else {  // n16 - c = 16
            uint32_t r16[16];
            tc::tmem_ld16(va + (uint32_t)c, r16);
            tc::tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const float v = __uint_as_float(r16[q]);
              vv = fmaf(v, v, vv);
            }
          }
        }
        // the mean columns (final: the last block barrier above follows every MMA of the tile)
        uint32_t rm[8];
        tc::tmem_ld8(va + (uint32_t)n16, rm);
        tc::tmem_wait_ld();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(bar(B_VE0 + vb));
        if (trd) trace_ev(p.trace, 17, 9, ti, trc);
        if (!dbl || vb == 0) ++vb0c;
        if (!dbl || vb == 1) ++vb1c;
        double mu_t = ((double)__uint_as_float(rm[0]) +
                       (double)__uint_as_float(rm[2]) * 4.8828125e-4) * (double)mun;
        const float a1_t = __uint_as_float(rm[1]) * mun;
        if (trd) trace_ev(p.trace, 18, 9, ti, trc);
        const float2 ri = rowinfo[(ti & 7u) * 128 + row];
        const uint32_t flags = __float_as_uint(ri.y);
        const int64_t rloc = (int64_t)(tile0 + kTs * tl) * 128 + row;
        const bool valid = (rloc < Ms) && !(flags & kFlagInvalid);
        const float u = 5.9604645e-8f;
        const float s2 = vv * vun2;
        const float var = fmaxf(sf2 - s2, 0.f);
        // K* relative error <= (dlog k / dh) dh + eval error; dh <= ~8 2^-22 (q^ + p^) for
        // the float16x3 augmented GEMM; margin x4
        // (+64: the float32 accumulation of the mean in the variance MMA, ~39 roundings)
        float dmu = (u * a1_t * (32.f * (ri.x + pmaxh) + 192.f) + dmu_abs) * p.bound_scale;
        if (mtier && rloc < Ms) {  // precise tier: the float64 mean (mean64.cu)
          mu_t = p.mean64[row0s + rloc];
          dmu = 1e-12f * a1_t * p.bound_scale;
        }
        const float dvar = vbk * (sf2 + s2) * p.bound_scale;
#ifndef GPBO_EXP_NOFINISH  // timing experiment only
        finish_fast(p, s, fs, thr, valid, row0s, rloc, mu_t, dmu, var, dvar,
                    (flags & kFlagUnsafe) != 0u, 2, 128, kDrainW0);
#else
        (void)dmu; (void)dvar; (void)valid; (void)rloc;
#endif
        if (trd) trace_ev(p.trace, 19, 9, ti, trc);
      }
    } else if (warp < kKWarps) {
      // ===================================================== K* warps
      // Per 64-wide panel q (= distance chunk q): part `part` of lane quarter lq evaluates
      // training points [64 q + kCW part, +kCW) for its 32 candidate rows: one tcgen05.ld of the
      // squared distances, K* = k(h), the float16 hi/lo split, tcgen05.st into the K* stage
      // (16-wide k steps kCW/16 part ..).
      const int lq = warp & 3, part = warp >> 2;
      const uint32_t tl_addr = tbase + ((uint32_t)(32 * lq) << 16);
      const int kind = m.kernel;
      const float c0 = m.c0, c1 = m.c1, c2 = m.c2, c3 = m.c3;
      uint32_t gk = gk_seg;
      uint32_t ec = gc_seg;  // distance chunk counter (= panel counter)
      int pp = 0;
      for (int g = 0; g < P; ++g) {
        const uint32_t st = ec % kDep;
        const int jb = 64 * pp + kCW * part;
        const int nv = min(kCW, n16 - jb);  // valid points of this warp (kCW, 16 or <= 0)
        const bool trw = (warp == 0 || warp == kKWarps - 1) && lane == 0;
        // kMerged (every search of the launch has n16 + 16 <= 128): one acquire for both
        // resources -- the distances (DF) and a free K* stage (KE) -- then one fence, and the
        // distance stage released together with the K* hand-over (config 3: -12 %).  Otherwise
        // separate acquires (the early DE release keeps the distance ring ahead).
        // A compile-time choice: the run-time branch cost registers and was slower in both cases.
        const uint32_t ks = gk % kKStages;
        const uint32_t da = tl_addr + kScr + 64u * st + (uint32_t)(kCW * part);
        uint32_t hr[kCW];
        auto load_h = [&]() {  // (a 16-point remainder: only its 16 columns)
          if (kCW == 32 && nv == 32) tc::tmem_ld32(da, hr);
          else tc::tmem_ld16(da, *reinterpret_cast<uint32_t(*)[16]>(hr));
          tc::tmem_wait_ld();
        };
        if (kMerged) {
          tc::mbar_wait(bar(B_DF0 + st), (ec / kDep) & 1u);
          tc::mbar_wait(bar(B_KE0 + ks), ((gk / kKStages) & 1u) ^ 1u);
          tc::tc_fence_after();
          if (nv > 0) load_h();
          if (trw) trace_ev(p.trace, 6, warp, gk, trc);
          if (trw) trace_ev(p.trace, 7, warp, gk, trc);
        } else {
          tc::mbar_wait(bar(B_DF0 + st), (ec / kDep) & 1u);
          if (trw) trace_ev(p.trace, 5, warp, gk, trc);
          tc::tc_fence_after();
          if (nv > 0) load_h();
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(bar(B_DE0 + st));  // the scratch stage is free
          ++ec;
          if (trw) trace_ev(p.trace, 6, warp, gk, trc);
          tc::mbar_wait(bar(B_KE0 + ks), ((gk / kKStages) & 1u) ^ 1u);
          tc::tc_fence_after();  // the V MMAs that read this K* stage have completed
          if (trw) trace_ev(p.trace, 7, warp, gk, trc);
        }
        // K* = k(h) for NE points, the float16 hi / lo split, and the stores of the NE / 16 k
        // steps (the 16-point remainder of a ragged last panel evaluates and stores only its own
        // 16 points: config 2 / 3 waste 7 / 12 % of the MUFU work otherwise)
        auto eval = [&](auto ne_tag) {
          constexpr int NE = decltype(ne_tag)::value;
          float kv[NE];
#ifdef GPBO_EXP_NOKSTAR  // timing experiment only: no kernel evaluation (wrong results)
          if (true) {
#pragma unroll
            for (int q = 0; q < NE; ++q) kv[q] = __uint_as_float(hr[q]);
          } else
#endif
          // |h| (a free source modifier) rather than max(h, 0): the GEMM-form h can be a few ulps
          // negative; |h| stays within the same error bound of the true h >= 0
          if (kind == GPBO_RBF) {
#pragma unroll
            for (int q = 0; q < NE; ++q)
              kv[q] = ex2_approx(fmaf(fabsf(__uint_as_float(hr[q])), c1, c0));
          } else {
#pragma unroll
            for (int q = 0; q < NE; ++q) {
              const float tq = sqrt_approx(fabsf(__uint_as_float(hr[q])));
              kv[q] = fmaf(tq, fmaf(tq, c3, c2), c0) * ex2_approx(tq * c1);
            }
          }
          uint32_t hw[NE / 2], lw[NE / 2];
#pragma unroll
          for (int q = 0; q < NE / 2; ++q) {
            const float h0 = __uint_as_float(__float_as_uint(kv[2 * q]) & 0xFFFFE000u);
            const float h1 = __uint_as_float(__float_as_uint(kv[2 * q + 1]) & 0xFFFFE000u);
            hw[q] = tc::pack_f16x2(h0, h1);
            lw[q] = tc::pack_f16x2(kv[2 * q] - h0, kv[2 * q + 1] - h1);
          }
          // this warp's k values are k steps (kCW / 16) part .. of the panel: hi at +8 per k
          // step, lo at +32
          const uint32_t kt = tl_addr + kKstar0 + 64u * ks + (uint32_t)(kCW / 2 * part);
          if constexpr (NE == 32) {
            tc::tmem_st16(kt, *reinterpret_cast<const uint32_t(*)[16]>(hw));
            tc::tmem_st16(kt + 32u, *reinterpret_cast<const uint32_t(*)[16]>(lw));
          } else {
            tc::tmem_st8(kt, *reinterpret_cast<const uint32_t(*)[8]>(hw));
            tc::tmem_st8(kt + 32u, *reinterpret_cast<const uint32_t(*)[8]>(lw));
          }
#ifndef GPBO_EXP_NOWAITST  // timing experiment only (races with the MMA)
          tc::tmem_wait_st();
#endif
        };
        if (nv > 0) {
          if (kCW == 32 && nv == 32) eval(std::integral_constant<int, kCW>());
          else eval(std::integral_constant<int, 16>());
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(bar(B_KF0 + ks));
        if (kMerged) {
          if (lane == 0) arrive_leader(bar(B_DE0 + st));  // the scratch stage is free
          ++ec;
        }
        if (trw) trace_ev(p.trace, 8, warp, gk, trc);
        ++gk;
        if (++pp == P64) pp = 0;
      }
    }
    gi += (uint32_t)T;
    gc_seg += (uint32_t)(T * ((npan + 1) >> 1));
    gk_seg += (uint32_t)P;  // (T * P64)
    ta = tb;
  }
  tc::tc_fence_before();
  // (pair: neither CTA leaves -- nor frees TMEM -- while the other may still arrive on its
  // barriers or be read by the MMAs)
  if (kPair) tc::cluster_sync();
  else __syncthreads();
#if defined(GPBO_TC_TRACE) || defined(GPBO_TC_CTATIME)  // per-CTA start / end (globaltimer, ns):
  // slice 5 of the trace buffer
  if (threadIdx.x == 0 && p.trace != nullptr && blockIdx.x < 8192) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    p.trace[5 * 16384 + 2 * blockIdx.x] = cta_t0;
    p.trace[5 * 16384 + 2 * blockIdx.x + 1] = t1;
  }
#endif
  if (warp == kDistW) {
    if (kPair) tc::tmem_dealloc2(tbase, kTmemCols);
    else tc::tmem_dealloc(tbase, kTmemCols);
  }
}

// ------------------------------------------------------------------ operand images (fit time)
__device__ double block_max_d(double v, double *red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r = fmax(r, red[i]);
  __syncthreads();
  return r;
}

// One CTA per search (several for one search: gridDim.y chunks share every loop), the body in
// score_pack.cuh (also run by the one-CTA fit kernel's tail, fit.cu).
__global__ void __launch_bounds__(256)
pack_tc_kernel(SearchMeta *meta, const double *Linv64, const double *Xs64, const double *alpha64,
               const float *ls32, unsigned char *img_all) {
  __shared__ double sc[5];
  __shared__ double il2[GPBO_MAX_D];
  asm volatile("griddepcontrol.launch_dependents;");  // the scoring kernel may start its setup
  pack_body(meta + blockIdx.x, meta[blockIdx.x], Linv64, Xs64, alpha64, ls32, img_all,
            blockIdx.y * blockDim.x + threadIdx.x, gridDim.y * blockDim.x, blockIdx.y == 0, sc,
            il2);
}

}  // namespace

static bool resident_fits(int n, int d) {
  const TcGeom g = tc_geom(n, d);
  if (g.n16 + kMeanRows > 256 || d + 2 > 64) return false;
  return tc_smem(g.img, g.kb, d).total <= kMaxSmem;
}

// the CTA-pair kernel (default; GPBO_TC_PAIR=0 selects the one-CTA kernel for A/B runs)
static bool pair_enabled() {
  static const bool on = [] {
    const char *e = getenv("GPBO_TC_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

// (the pair pays off only for the single-buffered V accumulator, n16 + 16 > 128: measured at
// config 2 fast phase 0.250 -> 0.244 ms, at config 3 -- two 64-wide panels per tile, double-
// buffered V -- 2.62 -> 2.92 ms: there the cross-SM handoffs outweigh the halved MMA issues)
bool tc_pair_fits(int n, int d) {
  if (!pair_enabled() || !resident_fits(n, d)) return false;
  const TcPairGeom g = tc_pair_geom(n, d);
  if (g.n16 + kMeanRows <= 128) return false;
  return tc_smem(g.half, g.kb, d).total <= kMaxSmem;
}

static bool stream_fits(int n, int d) {
  const TcsGeom g = tcs_geom(n, d);
  if (g.n16 > kTcsMaxN16 || d + 2 > 64) return false;
  return tcs_smem_bytes(g.kb, d) <= kMaxSmem;
}

bool tc_supported(const SearchMeta &m) { return m.tc_ok && !m.tc_stream; }
bool tcs_supported(const SearchMeta &m) { return m.tc_ok && m.tc_stream; }

int64_t tc_image_bytes(const SearchMeta &m) {
  if (m.tc_stream) return stream_fits(m.n, m.d) ? tcs_geom(m.n, m.d).img : 0;
  if (m.tc_pair) return 2 * (int64_t)tc_pair_geom(m.n, m.d).half;
  return resident_fits(m.n, m.d) ? tc_geom(m.n, m.d).img : 0;
}

// m.tc_stream on entry: 1 = streamed layout requested; it is also chosen when the resident
// image does not fit.  m.tc_pair on entry: 1 = CTA-pair layout requested (resident only).  (The
// caller makes both choices uniform over a model.)
void tc_fill_geometry(SearchMeta &m) {
  if (!resident_fits(m.n, m.d)) m.tc_stream = 1;
  if (m.tc_stream || !tc_pair_fits(m.n, m.d)) m.tc_pair = 0;
  if (m.tc_pair) {
    const TcPairGeom g = tc_pair_geom(m.n, m.d);
    m.n16 = g.n16;
    m.kb = g.kb;
    m.npan = (g.n16 + 31) / 32;
    m.img_bytes = g.half;  // per CTA of the pair (the model holds two halves)
    m.off_l = g.off_l;
    m.off_a = g.off_w;  // (no alpha pairs: the mean is MMA-accumulated)
    m.off_w = g.off_w;
  } else if (m.tc_stream) {
    const TcsGeom g = tcs_geom(m.n, m.d);
    m.n16 = g.n16;
    m.kb = g.kb;
    m.npan = g.npan;
    m.img_bytes = g.img;
    m.off_l = g.off_l;
    m.off_a = g.off_a;
    m.off_w = g.off_w;
  } else {
    const TcGeom g = tc_geom(m.n, m.d);
    m.n16 = g.n16;
    m.kb = g.kb;
    m.npan = g.npan;
    m.img_bytes = g.img;
    m.off_l = g.off_l;
    m.off_a = g.off_a;
    m.off_w = g.off_w;
  }
  m.tc_ok = tc_image_bytes(m) > 0;
}

bool tc_needs_stream(int n, int d) { return !resident_fits(n, d); }

cudaError_t launch_pack_tc(const SearchMeta *meta_d, int S, const double *Linv64,
                           const double *Xs64, const double *alpha64, const float *ls32,
                           unsigned char *img, cudaStream_t stream) {
  // 64 CTAs for one search (config 2: 18.8 -> 16.8 us, config 4: 45 -> 30 us), fewer per search
  // for large batches (config 3: 64 searches x 16)
#ifndef GPBO_PACK_PER
#define GPBO_PACK_PER 128  // measured: 64 -> 128 CTAs per search: config 2 pack 12.6 -> 11.0 us, config 4 26.8 -> 24.9; 256 same as 128
#endif
  const int per = std::max(4, std::min(GPBO_PACK_PER, 1024 / std::max(S, 1)));
  pack_tc_kernel<<<dim3(S, per), 256, 0, stream>>>(const_cast<SearchMeta *>(meta_d), Linv64, Xs64,
                                                   alpha64, ls32, img);
  return cudaGetLastError();
}

cudaError_t launch_score_tc(const ScoreLaunch &p, const SearchMeta *meta_h, int S,
                            int tile_lo, int total_tiles, int num_sms,
                            cudaStream_t stream) {
  int img_max = 0, kb_max = 1, d_max = 1;
  bool merged = true;  // every search double-buffers V (n16 + 16 <= 128)
  const bool pair = S > 0 && meta_h[0].tc_pair;  // (uniform over a model)
  for (int i = 0; i < S; ++i) {
    merged = merged && meta_h[i].n16 + kMeanRows <= 128;
    img_max = std::max(img_max, meta_h[i].img_bytes);
    kb_max = std::max(kb_max, meta_h[i].kb);
    d_max = std::max(d_max, meta_h[i].d);
  }
  const int smem = tc_smem(img_max, kb_max, d_max).total;
  if (smem > kMaxSmem) return cudaErrorInvalidValue;
  auto kern = pair ? (merged ? score_tc_kernel<true, true> : score_tc_kernel<false, true>)
                   : (merged ? score_tc_kernel<true, false> : score_tc_kernel<false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  // pair: clusters of two CTAs (one per SM of a TPC), total_tiles even (the host pads each
  // search to whole pair tiles)
  const int grid = pair ? 2 * std::max(1, std::min(num_sms / 2, total_tiles / 2))
                        : std::min(num_sms, total_tiles);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pair ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, p, tile_lo, total_tiles, img_max, kb_max, d_max);
}

}  // namespace gpbo
