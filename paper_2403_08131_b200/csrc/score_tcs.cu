// Fast phase of H6-H9 on the tcgen05 tensor cores for searches whose operand image does not fit
// in shared memory -- the large-n / large-d shapes (config 4: n = 500, d = 60; late config-5
// iterations: d = 35, n > ~150).  Same arithmetic as score_tc.cu (fp16x3 distance GEMM into TMEM,
// K* = k(h) on the CUDA cores into TMEM, triangular V = K* (L^-1)^T with A read from TMEM,
// s2~ = sf2 - sum V^2, EI bracket, threshold and refine list), but:
//   * the training operand (64-row chunks) and the L^-1 panels (slabs) are streamed from the
//     L2-resident image into shared-memory rings by TMA bulk copies (producer warp 13), in
//     exactly the order the two MMA issuers consume them;
//   * the V accumulator (256 TMEM columns) holds one 256-wide window of j at a time.  For
//     n16 > 256 a tile makes two passes: window 0 (j < 256) with K* panels 0..7, then window 1
//     (j >= 256) with all K* panels (panels 0..7 recomputed: +50 % K* work at n = 512, no
//     extra MMA work -- every (k, j >= k) block is multiplied exactly once).  The mean K* alpha
//     is accumulated in the last window, which sees every panel.
// Layout of the streamed image: score_tc.cuh.
//
// Warp roles (512 threads, one persistent CTA per SM):
//   warps 0-7   K* (2 warps per TMEM lane quarter, 16 columns of each panel each)
//   warps 8-11  drain (sum V_j^2 per window) + finish of the tile
//   warp 12     candidate loader (X* -> float16 hi/lo A operand)
//   warp 13     TMA producer of X chunks and L^-1 slabs (lane 0)
//   warp 14     TMEM allocator, small-image copy, distance MMA issuer
//   warp 15     variance MMA issuer
#include <cuda_fp16.h>

#include <algorithm>

#include "score_common.cuh"
#include "score_tc.cuh"
#include "score_tc_helpers.cuh"
#include "tc_prims.cuh"

namespace gpbo {

namespace {

constexpr int kThreads = 512;
constexpr uint32_t kTmemCols = 512;
constexpr int kMaxSmem = 227 * 1024;
constexpr int kDepth = 2;    // distance scratch stages (TMEM, 64 columns each)
constexpr int kKStages = 4;  // K* operand stages (TMEM, 32 columns each)
constexpr int kXSlots = 2;   // X chunk ring (shared memory)
constexpr int kLSlots = 2;   // L^-1 slab ring (shared memory)
constexpr uint32_t kScratch0 = 256;
constexpr uint32_t kKstar0 = 384;

enum {
  B_AF0 = 0, B_AF1, B_AE0, B_AE1,                          // candidate A tile (double buffer)
  B_DF0, B_DF1, B_DE0, B_DE1,                              // distance scratch ring
  B_KF0, B_KF1, B_KF2, B_KF3, B_KE0, B_KE1, B_KE2, B_KE3,  // K* stages
  B_VE,                                                    // V accumulator free (per window)
  B_VB0, B_VB1, B_VB2, B_VB3, B_VB4, B_VB5, B_VB6, B_VB7,  // V column block final (per window)
  B_SF,                                                    // raw candidate rows landed
  B_PF0, B_PF1, B_PE0, B_PE1,                              // partial sums K* -> drain
  B_XF0, B_XF1, B_XE0, B_XE1,                              // X chunk ring
  B_LF0, B_LF1, B_LE0, B_LE1,                              // L^-1 slab ring
  B_IMG, B_COUNT
};

enum : uint32_t { kFlagInvalid = 1u, kFlagUnsafe = 2u };

// dynamic shared memory: small image | A tiles x2 | staging | X ring | L ring | row info x8 |
// partials x2 | barriers
struct TcsSmem {
  int img, a, stage, xr, lr, rowinfo, part_mu, part_a1, bars, total;
};

__host__ __device__ inline TcsSmem tcs_smem(int kb_max, int d_max) {
  TcsSmem s;
  s.img = 0;
  s.a = tcs_align1k(kTcsMaxN16 * 8 + GPBO_MAX_D * 4);
  s.stage = s.a + 2 * kb_max * 8192;
  s.xr = tcs_align1k(s.stage + ((128 * d_max * 4 + 127) & ~127));
  s.lr = s.xr + kXSlots * kb_max * 4096;
  s.rowinfo = s.lr + kLSlots * kTcsSlabBytes;
  s.part_mu = s.rowinfo + 8 * 128 * 8;
  s.part_a1 = s.part_mu + 4 * 128 * 8;
  s.bars = s.part_a1 + 4 * 128 * 4;
  s.total = s.bars + B_COUNT * 8 + 16 + 1024;  // + tmem slot, + alignment slack
  return s;
}

__global__ void __launch_bounds__(kThreads, 1)
score_tcs_kernel(const ScoreLaunch p, int tile_lo, int total_tiles, int kb_max, int d_max) {
  extern __shared__ unsigned char sm_raw[];
  unsigned char *sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
  const TcsSmem L = tcs_smem(kb_max, d_max);
  unsigned char *simg = sm + L.img;
  unsigned char *Abuf = sm + L.a;
  float *stage = reinterpret_cast<float *>(sm + L.stage);
  unsigned char *xring = sm + L.xr;
  unsigned char *lring = sm + L.lr;
  float2 *rowinfo = reinterpret_cast<float2 *>(sm + L.rowinfo);
  double *part_mu = reinterpret_cast<double *>(sm + L.part_mu);
  float *part_a1 = reinterpret_cast<float *>(sm + L.part_a1);
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + L.bars);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + B_COUNT);
  auto bar = [&](int i) { return tc::smem_u32(bars + i); };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // this launch covers tiles [tile_lo, tile_lo + total_tiles) of the call (chunked host feeds)
  const int t0 = tile_lo + (int)((long long)total_tiles * blockIdx.x / gridDim.x);
  const int t1 = tile_lo + (int)((long long)total_tiles * (blockIdx.x + 1) / gridDim.x);

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(bar(B_AF0 + i), 32);
      tc::mbar_init(bar(B_AE0 + i), 1);
      tc::mbar_init(bar(B_PF0 + i), 8);
      tc::mbar_init(bar(B_PE0 + i), 4);
      tc::mbar_init(bar(B_DF0 + i), 1);
      tc::mbar_init(bar(B_DE0 + i), 8);
      tc::mbar_init(bar(B_XF0 + i), 1);
      tc::mbar_init(bar(B_XE0 + i), 1);
      tc::mbar_init(bar(B_LF0 + i), 1);
      tc::mbar_init(bar(B_LE0 + i), 1);
    }
    for (int i = 0; i < kKStages; ++i) {
      tc::mbar_init(bar(B_KF0 + i), 8);
      tc::mbar_init(bar(B_KE0 + i), 1);
    }
    tc::mbar_init(bar(B_VE), 4);
    for (int i = 0; i < 8; ++i) tc::mbar_init(bar(B_VB0 + i), 1);
    tc::mbar_init(bar(B_SF), 1);
    tc::mbar_init(bar(B_IMG), 1);
    tc::fence_mbar_init();
  }
  if (warp == 14) tc::tmem_alloc(tc::smem_u32(tmem_slot), kTmemCols);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  // programmatic dependent launch: barrier init and TMEM allocation above overlapped the
  // previous kernel (the operand pack); its outputs (meta constants, image) are read below.
  // The refine kernel may be scheduled on SMs this grid frees.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");

  // CTA-global counters (mbarrier phases continue across segments); every role advances the
  // ones it uses identically: tiles gi, distance chunks gc, K* items gk, window uses gv,
  // X slots gx, L slots gl, staging fills gs.
  uint32_t gi = 0, gc = 0, gk = 0, gv = 0, gx = 0, gl = 0, gsf = 0;
  uint32_t img_phase = 0;

  for (int ta = t0; ta < t1;) {
    const int s = search_of(p.tile_first, p.S, ta);
    const int tb = min(t1, p.tile_first[s + 1]);
    const SearchMeta &m = p.meta[s];
    __syncthreads();  // previous segment fully drained
    const int small_bytes = m.img_bytes - m.off_a;
    if (threadIdx.x == 448) {
      tc::mbar_arrive_expect_tx(bar(B_IMG), (uint32_t)small_bytes);
      tc::bulk_g2s(tc::smem_u32(simg), p.img + m.img_off + m.off_a, (uint32_t)small_bytes,
                   bar(B_IMG));
    }
    tc::mbar_wait(bar(B_IMG), img_phase);
    img_phase ^= 1u;
    const int n16 = m.n16, npan = m.npan, kb = m.kb;
    const int nw = (n16 + 255) / 256;
    const int np0 = tcs_window_panels(n16, 0);
    const int items = np0 + (nw == 2 ? npan : 0);              // K* panels per tile
    const int chunks = (np0 + 1) / 2 + (nw == 2 ? (npan + 1) / 2 : 0);  // distance chunks
    const int T = tb - ta;
    const int64_t Ms = p.m_off[s + 1] - p.m_off[s];
    const int tile0 = ta - p.tile_first[s];
    const unsigned char *gimg = p.img + m.img_off;

    if (warp == 13) {
      // ===================================================== TMA producer (lane 0)
      if (lane == 0) {
        uint32_t cx = gx, cl = gl;
        const uint32_t xbytes = (uint32_t)kb * 4096u;
        for (int tl = 0; tl < T; ++tl) {
          int loff = m.off_l;
          for (int w = 0; w < nw; ++w) {
            const int npw = tcs_window_panels(n16, w);
            for (int pp = 0; pp < npw; ++pp) {
              if ((pp & 1) == 0) {  // the chunk of panels pp, pp + 1
                const uint32_t xs = cx % kXSlots;
                tc::mbar_wait(bar(B_XE0 + xs), ((cx / kXSlots) & 1u) ^ 1u);
                tc::mbar_arrive_expect_tx(bar(B_XF0 + xs), xbytes);
                tc::bulk_g2s(tc::smem_u32(xring + xs * xbytes), gimg + (size_t)(pp >> 1) * xbytes,
                             xbytes, bar(B_XF0 + xs));
                ++cx;
              }
              const uint32_t ls = cl % kLSlots;
              const uint32_t lbytes = (uint32_t)tcs_slab_rows(n16, w, pp) * 128u;
              tc::mbar_wait(bar(B_LE0 + ls), ((cl / kLSlots) & 1u) ^ 1u);
              tc::mbar_arrive_expect_tx(bar(B_LF0 + ls), lbytes);
              tc::bulk_g2s(tc::smem_u32(lring + ls * kTcsSlabBytes), gimg + loff, lbytes,
                           bar(B_LF0 + ls));
              loff += (int)lbytes;
              ++cl;
            }
          }
        }
      }
      __syncwarp();
    } else if (warp == 14) {
      // ===================================================== distance MMA issuer
      const uint32_t H32 = tc::sdesc_hi(32);
      const uint32_t abase = tc::sdesc_lo(tc::smem_u32(Abuf));
      const uint32_t xb0 = tc::sdesc_lo(tc::smem_u32(xring));
      uint32_t cc = gc, cx = gx;
      for (int tl = 0; tl < T; ++tl) {
        const uint32_t ti = gi + tl, ab = ti & 1u;
        tc::mbar_wait(bar(B_AF0 + ab), (ti >> 1) & 1u);
        tc::tc_fence_after();
        for (int w = 0; w < nw; ++w) {
          const int nq = (tcs_window_panels(n16, w) + 1) / 2;
          for (int q = 0; q < nq; ++q) {
            const uint32_t d_st = cc % kDepth, xs = cx % kXSlots;
            tc::mbar_wait(bar(B_DE0 + d_st), ((cc / kDepth) & 1u) ^ 1u);
            tc::mbar_wait(bar(B_XF0 + xs), (cx / kXSlots) & 1u);
            tc::tc_fence_after();
            const uint32_t idn = tc::idesc_f16((uint32_t)min(64, n16 - 64 * q));
            const uint32_t dt = tbase + kScratch0 + 64u * d_st;
            uint32_t a = abase + ab * (uint32_t)kb * 512u;  // 8192 B per K block
            uint32_t bq = xb0 + xs * (uint32_t)kb * 256u;   // kb x 4096 B per slot
            for (int k = 0; k < kb; ++k) {
              tc::mma_f16_split(dt, a, H32, bq, H32, idn, k > 0);
              tc::mma_f16_split(dt, a, H32, bq + 128u, H32, idn, 1u);         // B lo: +2048 B
              tc::mma_f16_split(dt, a + 256u, H32, bq, H32, idn, 1u);         // A lo: +4096 B
              a += 512u;
              bq += 256u;
            }
            tc::mma_commit_warp(bar(B_DF0 + d_st));
            tc::mma_commit_warp(bar(B_XE0 + xs));
            ++cc;
            ++cx;
          }
        }
        tc::mma_commit_warp(bar(B_AE0 + ab));  // A tile consumed
      }
      __syncwarp();
    } else if (warp == 15) {
      // ===================================================== variance MMA issuer
      const uint32_t H64 = tc::sdesc_hi(64);
      const uint32_t lb0 = tc::sdesc_lo(tc::smem_u32(lring));
      uint32_t ck = gk, cl = gl, cv = gv;
      for (int tl = 0; tl < T; ++tl) {
        for (int w = 0; w < nw; ++w) {
          const int wlo = 256 * w, wend = tcs_window_end(n16, w);
          const int npw = tcs_window_panels(n16, w);
          const int nblk = (wend - wlo + 31) / 32;
          tc::mbar_wait(bar(B_VE), (cv & 1u) ^ 1u);  // the drain has read the previous window
          tc::tc_fence_after();
          for (int pp = 0; pp < npw; ++pp) {
            const uint32_t ks = ck % kKStages, ls = cl % kLSlots;
            tc::mbar_wait(bar(B_KF0 + ks), (ck / kKStages) & 1u);
            tc::mbar_wait(bar(B_LF0 + ls), (cl / kLSlots) & 1u);
            tc::tc_fence_after();
            const int r0 = max(wlo, 32 * pp);
            const int R = wend - r0;
            const uint32_t kt = tbase + kKstar0 + 32u * ks;
            const uint32_t slab = lb0 + ls * (uint32_t)(kTcsSlabBytes >> 4);
            const uint32_t R16 = (uint32_t)R * 4u;  // R * 64 B >> 4: hi -> lo
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int js = max(wlo, 32 * pp + 16 * h);
              if (js < wend) {
                const uint32_t idn = tc::idesc_f16((uint32_t)(wend - js));
                const uint32_t dt = tbase + (uint32_t)(js - wlo);
                const uint32_t ka = kt + 8u * h;  // k step h: hi at +8h, lo at +16 + 8h
                const uint32_t lb = slab + (uint32_t)(js - r0) * 4u + 2u * h;  // rows, +32 B k
                tc::mma_f16_ts(dt, ka, lb, H64, idn, (pp | h) ? 1u : 0u);
                tc::mma_f16_ts(dt, ka, lb + R16, H64, idn, 1u);
                tc::mma_f16_ts(dt, ka + 16u, lb, H64, idn, 1u);
              }
            }
            tc::mma_commit_warp(bar(B_KE0 + ks));
            tc::mma_commit_warp(bar(B_LE0 + ls));
            // V block b = pp - 8 w of the window receives no later contribution
            if (32 * pp >= wlo) tc::mma_commit_warp(bar(B_VB0 + (pp - 8 * w)));
            ++ck;
            ++cl;
          }
          // every block barrier completes once per window
          for (int b = nblk; b < 8; ++b) tc::mma_commit_warp(bar(B_VB0 + b));
          ++cv;
        }
      }
      __syncwarp();
    } else if (warp == 12) {
      // ===================================================== candidate loader (32 threads)
      const int d = m.d;
      const float *wsc = reinterpret_cast<const float *>(simg + (m.off_w - m.off_a));
      uint32_t cs = gsf;
      for (int tl = 0; tl < T; ++tl) {
        const uint32_t ti = gi + tl, ab = ti & 1u;
        const int64_t row0 = (int64_t)(tile0 + tl) * 128;
        const int rows = (int)(Ms - row0 < 128 ? Ms - row0 : 128);
        {  // fetch the raw rows of this tile into the staging buffer
          const float *src = p.Xstar + p.x_off[s] + row0 * d;
          const uint32_t bytes = (uint32_t)(rows * d * 4);
          if ((((uintptr_t)src) & 15u) == 0 && (bytes & 15u) == 0) {
            if (lane == 0) {
              tc::mbar_arrive_expect_tx(bar(B_SF), bytes);
              tc::bulk_g2s(tc::smem_u32(stage), src, bytes, bar(B_SF));
            }
          } else {
            for (int e = lane; e < rows * d; e += 32) stage[e] = __ldg(src + e);
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(bar(B_SF));
          }
        }
        tc::mbar_wait(bar(B_SF), cs & 1u);
        ++cs;
        tc::mbar_wait(bar(B_AE0 + ab), ((ti >> 1) & 1u) ^ 1u);
        const uint32_t a0 = tc::smem_u32(Abuf) + ab * kb * 8192;
        for (int r = lane; r < 128; r += 32) {
          const bool valid = r < rows;
#ifndef GPBO_LOADER_SCALAR  // (A/B switch)
          if ((d & 3) == 0) {  // vectorised path (config 4)
            float qh;
            bool nan;
            convert_row_vec4(stage, wsc, r, d, kb, valid, a0, qh, nan);
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
              const float x = stage[r * d + c];
              nan |= !isfinite(x);
              const float v = x * wsc[c];
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
                  if (c < d) v = stage[r * d + c] * wsc[c];
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
        __syncwarp();  // staging free (next fetch), A tile complete
        tc::mbar_arrive(bar(B_AF0 + ab));
      }
    } else if (warp >= 8 && warp < 12) {
      // ===================================================== drain + finish (warps 8-11)
      const int lq = warp & 3;
      const int row = 32 * lq + lane;
      const uint32_t va = tbase + ((uint32_t)(32 * lq) << 16);
      const FinishSeg fs = finish_seg(p, s);
      const int64_t row0s = p.m_off[s];
      const float vun2 = m.vunscale2, sf2 = m.sf2, pmaxh = m.pmax_h, lrs = m.linv_rowsum;
      const int nn = m.n;
      const bool mtier = p.mean64 != nullptr && m.mean_tier;  // precise-mean tier (mean64.cu)
      // variance bound 4 var_bound(u, sf2, s2, n, lrs) = vbk (sf2 + s2), its factor hoisted
      const float vbk = 4.f * 16.f * 5.9604645e-8f * sqrtf((float)nn) * (1.f + 0.01f * lrs * sqrtf(sf2));
      uint32_t cv = gv;
      for (int tl = 0; tl < T; ++tl) {
        const uint32_t ti = gi + tl;
        const float thr = p.mode == kModeArgmax ? read_thr(p, s) : 0.f;
        float vv = 0.f;
        for (int w = 0; w < nw; ++w) {
          const int width = tcs_window_end(n16, w) - 256 * w;
          const int nblk = (width + 31) / 32;
          for (int b = 0; b < nblk; ++b) {
            tc::mbar_wait(bar(B_VB0 + b), cv & 1u);
            tc::tc_fence_after();
            const int c = 32 * b;
            if (c + 32 <= width) {
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
            } else {  // 16 columns
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
          // blocks nblk..7 complete too (committed by the issuer): consume their phase
          for (int b = nblk; b < 8; ++b) tc::mbar_wait(bar(B_VB0 + b), cv & 1u);
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(bar(B_VE));
          ++cv;
        }
        const uint32_t par = ti & 1u;
        tc::mbar_wait(bar(B_PF0 + par), (ti >> 1) & 1u);
        double mu_t = part_mu[par * 128 + row] + part_mu[(2 + par) * 128 + row];
        const float a1_t = part_a1[par * 128 + row] + part_a1[(2 + par) * 128 + row];
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(bar(B_PE0 + par));
        const float2 ri = rowinfo[(ti & 7u) * 128 + row];
        const uint32_t flags = __float_as_uint(ri.y);
        const int64_t rloc = (int64_t)(tile0 + tl) * 128 + row;
        const bool valid = (rloc < Ms) && !(flags & kFlagInvalid);
        const float u = 5.9604645e-8f;
        const float s2 = vv * vun2;
        const float var = fmaxf(sf2 - s2, 0.f);
        // error bounds as in score_tc.cu
        float dmu = u * a1_t * (32.f * (ri.x + pmaxh) + 128.f) * p.bound_scale;
        if (mtier && rloc < Ms) {  // precise tier: the float64 mean (mean64.cu)
          mu_t = p.mean64[row0s + rloc];
          dmu = 1e-12f * a1_t * p.bound_scale;
        }
        const float dvar = vbk * (sf2 + s2) * p.bound_scale;
        finish_fast(p, s, fs, thr, valid, row0s, rloc, mu_t, dmu, var, dvar,
                    (flags & kFlagUnsafe) != 0u, 2, 128, 8);
      }
    } else if (warp < 8) {
      // ===================================================== K* warps (0-7)
      const int lq = warp & 3, half = warp >> 2;
      const int row = 32 * lq + lane;
      const uint32_t tl_addr = tbase + ((uint32_t)(32 * lq) << 16);
      const float2 *ap = reinterpret_cast<const float2 *>(simg);
      const int kind = m.kernel;
      const float c0 = m.c0, c1 = m.c1, c2 = m.c2, c3 = m.c3;
      uint32_t ck = gk, ec = gc;
      const int P = T * items;
      double mu = 0.0;
      float a1 = 0.f;
      int tl = 0, w = 0, pp = 0;
      int npw = np0;
      uint32_t hbuf[2][16];
      auto load_dist = [&](int ppn, uint32_t chunk, uint32_t (&dst)[16]) {
        const uint32_t st = chunk % kDepth;
        tc::mbar_wait(bar(B_DF0 + st), (chunk / kDepth) & 1u);
        tc::tc_fence_after();
        if (32 * ppn + 16 * half < n16)
          tc::tmem_ld16(tl_addr + kScratch0 + 64u * st + 32u * (ppn & 1) + 16u * half, dst);
      };
      auto step = [&](int g, uint32_t (&hr)[16], uint32_t (&nx)[16]) {
        const uint32_t st = ec % kDepth;
        const int jb = 32 * pp + 16 * half;
        const bool active = jb < n16;
        const bool last_window = w == nw - 1;
        tc::tmem_wait_ld();
        tc::tc_fence_before();
        __syncwarp();
        if ((pp & 1) || pp == npw - 1) {  // both panels of the chunk loaded: free the stage
          if (lane == 0) tc::mbar_arrive(bar(B_DE0 + st));
          ++ec;
        }
        // position of item g + 1
        int nw_ = w, np_ = pp + 1, npw_ = npw;
        if (np_ == npw) {
          np_ = 0;
          nw_ = w + 1 == nw ? 0 : w + 1;
          npw_ = tcs_window_panels(n16, nw_);
        }
        if (g + 1 < P) load_dist(np_, ec, nx);
        const uint32_t ks = ck % kKStages;
        tc::mbar_wait(bar(B_KE0 + ks), ((ck / kKStages) & 1u) ^ 1u);
        tc::tc_fence_after();
        float muf = 0.f, a1f = 0.f;
        if (active) {
          float kv[16];
          if (kind == GPBO_RBF) {
#pragma unroll
            for (int q = 0; q < 16; ++q)
              kv[q] = ex2_approx(fmaf(fabsf(__uint_as_float(hr[q])), c1, c0));
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const float tq = sqrt_approx(fabsf(__uint_as_float(hr[q])));
              kv[q] = fmaf(tq, fmaf(tq, c3, c2), c0) * ex2_approx(tq * c1);
            }
          }
          if (last_window) {
            const float4 *ap4 = reinterpret_cast<const float4 *>(ap + jb);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 a = ap4[q];
              muf = fmaf(kv[2 * q], a.x, muf);
              a1f = fmaf(kv[2 * q], a.y, a1f);
              muf = fmaf(kv[2 * q + 1], a.z, muf);
              a1f = fmaf(kv[2 * q + 1], a.w, a1f);
            }
          }
          uint32_t hw[8], lw[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float h0 = __uint_as_float(__float_as_uint(kv[2 * q]) & 0xFFFFE000u);
            const float h1 = __uint_as_float(__float_as_uint(kv[2 * q + 1]) & 0xFFFFE000u);
            hw[q] = tc::pack_f16x2(h0, h1);
            lw[q] = tc::pack_f16x2(kv[2 * q] - h0, kv[2 * q + 1] - h1);
          }
          const uint32_t kt = tl_addr + kKstar0 + 32u * ks + 8u * half;
          tc::tmem_st8(kt, hw);
          tc::tmem_st8(kt + 16u, lw);
          tc::tmem_wait_st();
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(bar(B_KF0 + ks));
        ++ck;
        mu += (double)muf;
        a1 += a1f;
        const bool tile_done = np_ == 0 && nw_ == 0;
        w = nw_;
        pp = np_;
        npw = npw_;
        if (tile_done) {  // hand the partial sums to the drain warps
          const uint32_t ti = gi + tl, par = ti & 1u;
          tc::mbar_wait(bar(B_PE0 + par), ((ti >> 1) & 1u) ^ 1u);
          part_mu[(2 * half + par) * 128 + row] = mu;
          part_a1[(2 * half + par) * 128 + row] = a1;
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(bar(B_PF0 + par));
          mu = 0.0;
          a1 = 0.f;
          ++tl;
        }
      };
      if (P > 0) load_dist(0, ec, hbuf[0]);
      for (int g = 0; g < P; g += 2) {
        step(g, hbuf[0], hbuf[1]);
        if (g + 1 < P) step(g + 1, hbuf[1], hbuf[0]);
      }
    }
    gi += (uint32_t)T;
    gc += (uint32_t)(T * chunks);
    gk += (uint32_t)(T * items);
    gv += (uint32_t)(T * nw);
    gx += (uint32_t)(T * chunks);
    gl += (uint32_t)(T * items);
    gsf += (uint32_t)T;
    ta = tb;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 14) tc::tmem_dealloc(tbase, kTmemCols);
}

}  // namespace

int tcs_smem_bytes(int kb_max, int d_max) { return tcs_smem(kb_max, d_max).total; }

cudaError_t launch_score_tcs(const ScoreLaunch &p, const SearchMeta *meta_h, int S,
                             int tile_lo, int total_tiles, int num_sms,
                            cudaStream_t stream) {
  int kb_max = 1, d_max = 1;
  for (int i = 0; i < S; ++i) {
    kb_max = std::max(kb_max, meta_h[i].kb);
    d_max = std::max(d_max, meta_h[i].d);
  }
  const int smem = tcs_smem(kb_max, d_max).total;
  if (smem > kMaxSmem) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(score_tcs_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int grid = std::min(num_sms, total_tiles);
  // programmatic dependent launch after the operand pack (the kernel's griddepcontrol.wait
  // precedes every read of the image), as score_tc
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, score_tcs_kernel, p, tile_lo, total_tiles, kb_max, d_max);
}

}  // namespace gpbo
