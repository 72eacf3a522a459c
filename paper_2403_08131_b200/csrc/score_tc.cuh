// tcgen05 scoring path: envelope, operand-image geometry, launchers (see score_tc.cu and
// score_tcs.cu).
#pragma once
#include "gpbo_internal.cuh"

namespace gpbo {
constexpr int kTcTile = 128;

// ---- streamed layout (score_tcs.cu): for searches whose operand image does not fit in shared
// memory (n16 > 256, or large d).  The training operand and L^-1 stay in global memory (L2
// resident) and are streamed through shared-memory rings by TMA bulk copies.  The V accumulator
// (TMEM, 256 columns) covers the columns j of one 256-wide window at a time: window w holds
// j in [256 w, min(n16, 256 (w + 1))) and needs the K* panels p with 32 p < window end.
// Image (bytes from img_off):
//   [0, off_l)       X chunks: chunk q = training rows [64 q, 64 q + 64), per 16-wide K block
//                    a float16 hi (2048 B) and lo (2048 B) block, SWIZZLE_32B K-major
//   [off_l, off_a)   L^-1 slabs in consumption order (window 0 panels, then window 1 panels):
//                    rows j in [max(256 w, 32 p), min(n16, 256 (w + 1))), k in [32 p, 32 p + 32)
//                    as float16 hi (R x 64 B) then lo (R x 64 B), SWIZZLE_64B K-major
//   [off_a, off_w)   alpha pairs (alpha', |alpha'|) float32, n16 entries
//   [off_w, img)     per-dimension candidate scales (GPBO_MAX_D floats)
// [off_a, img) is the small per-search part copied to shared memory once per segment.
constexpr int kTcsMaxN16 = 512;
constexpr int kTcsSlabBytes = 256 * 128;  // largest L^-1 slab (256 rows x 32 k x hi/lo)

struct TcsGeom {
  int n16, kb, npan, nw, np0, nchunk, off_l, off_a, off_w, img;
};

__host__ __device__ inline int tcs_align1k(int v) { return (v + 1023) & ~1023; }

__host__ __device__ inline int tcs_window_end(int n16, int w) {
  return n16 < 256 * (w + 1) ? n16 : 256 * (w + 1);
}
// panels of window w (all panels with 32 p < window end)
__host__ __device__ inline int tcs_window_panels(int n16, int w) {
  return (tcs_window_end(n16, w) + 31) / 32;
}
__host__ __device__ inline int tcs_slab_rows(int n16, int w, int p) {
  const int r0 = 256 * w > 32 * p ? 256 * w : 32 * p;
  return tcs_window_end(n16, w) - r0;
}

__host__ __device__ inline TcsGeom tcs_geom(int n, int d) {
  TcsGeom g;
  g.n16 = (n + 15) & ~15;
  g.kb = (d + 2 + 15) / 16;
  g.npan = (g.n16 + 31) / 32;
  g.nw = (g.n16 + 255) / 256;
  g.np0 = tcs_window_panels(g.n16, 0);
  g.nchunk = (g.n16 + 63) / 64;
  g.off_l = tcs_align1k(g.nchunk * g.kb * 4096);
  int lbytes = 0;
  for (int w = 0; w < g.nw; ++w)
    for (int p = 0; p < tcs_window_panels(g.n16, w); ++p) lbytes += tcs_slab_rows(g.n16, w, p) * 128;
  g.off_a = tcs_align1k(g.off_l + lbytes);
  g.off_w = g.off_a + g.n16 * 8;
  g.img = tcs_align1k(g.off_w + GPBO_MAX_D * 4);
  return g;
}

// Fills the tcgen05 geometry fields of m (n16, kb, npan, image offsets, tc_ok) from n, d and
// m.tc_stream (the layout chosen at fit time).
void tc_fill_geometry(SearchMeta &m);
// The resident (shared-memory image) kernel covers m / the streamed kernel covers m.
bool tc_supported(const SearchMeta &m);
bool tcs_supported(const SearchMeta &m);
int64_t tc_image_bytes(const SearchMeta &m);
cudaError_t launch_pack_tc(const SearchMeta *meta_d, int S, const double *Linv64,
                           const double *Xs64, const double *alpha64, const float *ls32,
                           unsigned char *img, cudaStream_t stream);
// Tiles [tile_lo, tile_lo + total_tiles) of the call (tile indices as in p.tile_first).
cudaError_t launch_score_tc(const ScoreLaunch &p, const SearchMeta *meta_h, int S, int tile_lo,
                            int total_tiles, int num_sms, cudaStream_t stream);
cudaError_t launch_score_tcs(const ScoreLaunch &p, const SearchMeta *meta_h, int S, int tile_lo,
                             int total_tiles, int num_sms, cudaStream_t stream);
int tcs_smem_bytes(int kb_max, int d_max);
// true when the resident image of an (n, d) search does not fit in shared memory
bool tc_needs_stream(int n, int d);
// the CTA-pair resident layout (score_tc.cu kPair) covers an (n, d) search
bool tc_pair_fits(int n, int d);
}  // namespace gpbo
