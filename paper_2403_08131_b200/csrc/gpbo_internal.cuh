// Internal device/host definitions shared by the libgpbo CUDA translation units.
// Nothing here is shared with oracle/ (the oracle is independent Python).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/gpbo.h"
#include "../../include/gpbo_test.h"

namespace gpbo {

#ifndef GPBO_FIT_THREADS
#define GPBO_FIT_THREADS 384
#endif
constexpr int kFitThreads = GPBO_FIT_THREADS;
constexpr int kSimtTile = 64;  // candidates per CTA of the CUDA-core scoring kernel
// Panel width of the fit's blocked factorisation (fit.cu) and its shared-memory plan:
// y~, w (n-vectors), spare/flags, the block maps M, N, R, 2 x 8 panel rows G of stride gs (a
// pair of panels), and -- for
// n <= kFitSmemMaxN -- the working matrix as the lower triangle of 8 x 8 tiles, each row-major
// (27 * 28 / 2 tiles * 512 B = 189 KB at n = 216).
constexpr int kFitB = 8;
constexpr int kFitSmemMaxN = 216;
constexpr int kFitSmemBudget = 227 * 1024 - 512;  // dynamic shared memory of the fit kernel
__host__ __device__ constexpr int fit_nr8(int n) { return (n + 7) & ~7; }
// G row stride (doubles) = GPBO_GS_MOD (mod 16).  A DMMA fragment load of G reads rows tig = 0..3
// at columns gid; 64-bit loads are served per half-warp (lanes 4 gid + tig, gid < 4), so the
// rows must land in distinct 4-double bank groups: 4 (mod 16) does that, 8 (mod 16) pairs rows
// 0 / 2 and 1 / 3 on the same banks (2-way conflicts)
#ifndef GPBO_GS_MOD
#define GPBO_GS_MOD 4
#endif
__host__ __device__ constexpr int fit_gstride(int n) { return ((n + 15) & ~15) + GPBO_GS_MOD; }
__host__ __device__ constexpr int fit_tile_doubles(int n) {
  return ((n + 7) / 8) * ((n + 7) / 8 + 1) / 2 * 64;
}
__host__ __device__ constexpr int fit_smem_doubles(int n, bool in_smem) {
  return 2 * fit_nr8(n) + 24 + 3 * 64 + 16 * fit_gstride(n) + (in_smem ? fit_tile_doubles(n) : 0);
}

// Per-search state of a fitted model (device copy in gpbo_model::meta_d, host copy in meta_h).
struct SearchMeta {
  int32_t n, d;         // observations, encoded dims
  int32_t n_pad, d_pad; // n rounded up to 64 (scoring operand), d rounded up to 8
  int32_t kernel;       // gpbo_kernel
  float sf2, sn2;       // signal / noise variance (standardised units)
  int64_t x_off;        // raw X  (float32, n x d)            into model.X32
  int64_t ls_off;       // lengthscales (float32, d)          into model.ls32
  int64_t y_off;        // y (float64, n)                     into model.y64
  int64_t mat_off;      // n x n float64: L col-major, L^-1 row-major  into model.L64 / .Linv64
  int64_t xs_off;       // X/l (float32, n_pad x d_pad)       into model.Xs32
  int64_t lt_off;       // (L^-1)^T float32 n_pad x n_pad      into model.LT32
  int64_t a_off;        // alpha (n_pad)                      into model.alpha64
  int64_t img_off;      // tcgen05 operand image (bytes)      into model.img
  // fit results
  double mean, std, best, alpha_l1;
  double lml;           // log marginal likelihood of y~ (standardised), -inf if the fit failed
  int32_t mean_tier;    // 1: precise mean tier (mean64.cu), chosen at fit time (reading R13)
  float pmax;           // max_j |x_j / l|^2 (error-bound input of the fast phase)
  float alpha_max;      // max_j |alpha_j|
  float linv_rowsum;    // max_j sum_k |(L^-1)_jk| (variance error-bound input)
  double linv_absmax;   // max |(L^-1)_jk| (operand scaling of the tcgen05 image)
  // ---- tcgen05 fast phase (score_tc.cu); valid when tc_ok
  int32_t tc_ok;
  int32_t tc_stream;    // streamed image layout (score_tcs.cu) instead of the resident one
  int32_t tc_pair;      // resident CTA-pair layout (two half images, score_tc.cu kPair)
  int32_t n16;          // n rounded up to 16 (V accumulator columns)
  int32_t kb;           // 16-wide K blocks of the augmented distance operand [x, |x|^2, 1]
  int32_t npan;         // 32-wide training-point panels
  int32_t img_bytes;    // operand image bytes (shared-memory resident per search)
  int32_t off_l, off_a, off_w;  // byte offsets of L^-1 panels, alpha pairs, candidate scales
  float c0, c1, c2, c3; // kernel-value constants in the scaled MMA units (see pack_tc)
  float hscale;         // true h = MMA h * hscale
  float vunscale2;      // |v|^2 = sum of squared V accumulator * vunscale2
  float munscale;       // mu~ = (V[n16] + V[n16 + 2] 2^-11) * munscale (mean rows of the image)
  float pmax_h;         // max_j p^_j in true h units (error-bound input)
  double jitter;
  int32_t jitter_k;
  int32_t status;       // gpbo_status of this search
  int32_t use_smem;     // fit keeps its working matrix in shared memory
  int32_t xs_smem;      // fit stages x / l (n x d float64) in shared memory for the Gram
  int64_t scr_off;      // else: its tile-packed working matrix (fit_tile_doubles) in model.Wscr64
  int64_t kt_off;       // kernel matrix k(X, X) without noise / jitter, tile-packed, in model.Kt64
  int64_t stg_off;      // cluster fit: the panel's G rows staged in global memory for the
                        // multicast bulk copies (2 x 8 fit_nr8(n) doubles) in model's G64
};

// Candidate flagged by the fast phase for the float64 refine phase.  The refine re-scores it in
// float64 and checks the fast phase's bracket ei_lo <= EI <= ei_hi (the argmax filter's
// soundness); a violation re-scores the whole search exactly (api.cu, argmax_tail).
struct RefineEntry {
  uint32_t s;     // search (launch-relative) | kEntryAudit
  uint32_t row;   // local candidate row
  float ei_lo;    // lower bound of EI~ from the fast phase (0 when not evaluated)
  float ei_hi;    // upper bound of EI~ from the fast phase
};
// Audit entry: a candidate the fast phase did NOT flag, sampled deterministically (1 in 2^14 by
// a multiplicative hash of its global index: (u32)(gidx * 0x9E3779B1) >> kAuditShift == 0) so the
// refine also checks the upper bound that excluded it; never skipped by the threshold test.
constexpr uint32_t kEntryAudit = 0x80000000u;
constexpr uint32_t kAuditShift = 18;

enum ScoreMode : int32_t {
  kModeArgmax = 0,     // fast phase flags candidates, refine computes the final keys
  kModePosterior = 1,  // fast phase writes var~ of every candidate, refine writes mu/var/ei
  kModeDebug = 2       // fast phase writes its own mu32 / dmu / EI bounds (tests)
};

// One scoring launch covers several searches; tile t of the launch belongs to search
// tile_search[t], local tile index t - tile_first[search].
struct ScoreLaunch {
  const SearchMeta *meta;
  const float *Xstar;          // concatenated candidate rows
  const int64_t *m_off;        // [S+1] candidate row offsets (device copy)
  const int64_t *m_base;       // [S] global index of the first local row
  const int64_t *x_off;        // [S] element offset of search s's first row in Xstar
  const double *best;          // [S] standardised incumbent
  const int32_t *tile_first;   // [S+1] prefix sums of tiles per search
  int32_t S;
  const float *Xs32;
  const float *LT32;
  const double *alpha64;
  const float *ls32;
  const unsigned char *img;    // tcgen05 operand images
  unsigned long long *keys;    // [S] per-search argmax keys (atomicMax)
  float *out_mu, *out_var, *out_ei;  // optional per-candidate outputs (raw units)
  int32_t mode;                // ScoreMode
  unsigned int *thr;           // [S] float bits of the running max EI_lo (argmax mode)
  RefineEntry *list;           // refine list (argmax mode)
  unsigned int *list_count;
  uint32_t list_cap;
  float *dbg_mu, *dbg_dmu, *dbg_var, *dbg_dvar, *dbg_eilo, *dbg_eihi;  // debug mode
  unsigned long long *trace;   // optional clock64 event trace of CTA 0 (gpbo_debug_trace)
  const double *mean64;        // precise-tier float64 mean per launch row (NULL: none)
  float bound_scale;           // error-bound multiplier: 1 (test hook gpbo_debug_bound_scale)
  int32_t break_bracket;       // test hook: halve every EI bracket (deliberately unsound)
};

// Float64 refine phase (refine.cu).
struct RefineLaunch {
  const SearchMeta *meta;
  const float *Xstar;
  const int64_t *m_off, *m_base, *x_off;
  const double *best;
  const double *Xs64;          // X / l in float64, n x d per search (indexed by x_off)
  const float *ls32;
  const double *alpha64;
  const double *Linv64;        // L^-1, n x n row-major per search (mat_off), lower part
  unsigned long long *keys;
  const unsigned int *thr;
  const RefineEntry *list;     // argmax mode: entries; posterior mode: NULL (dense rows)
  const unsigned int *list_count;
  int32_t dense_s;             // posterior mode: search index
  int64_t dense_rows;          // posterior mode: number of rows
  const float *dense_var;      // posterior mode: var~ per row from the fast phase
  float *out_mu, *out_var, *out_ei;
  int32_t dense_keys;          // dense mode: argmax keys of every row instead of outputs
  unsigned long long *viol;    // [S] bracket violations found by the refine (argmax mode)
};

}  // namespace gpbo

// Kernel launchers (defined in the .cu files).
namespace gpbo {
// Fit kernel inputs (the caller's arrays, host-staged or device) and the model arrays it fills.
struct FitIO {
  const float *X_src, *ls_src;   // [sum n_s d_s], [sum d_s]
  const double *y_src;           // [sum n_s]
  const float *sf2_src, *sn2_src;  // [S] (device); null: taken from the meta records
  float *X32, *ls32;             // model copies (skipped when equal to the sources)
  double *y64, *L64, *Linv64, *Xs64, *alpha64, *Wscr64;
  double *Kt64;                  // the Gram pre-pass output (tile-packed, no noise / jitter)
  double *pm_part;               // [16 S] per-CTA max |x / l|^2 of the pre-pass
  double *G64;                   // cluster fit staging (SearchMeta::stg_off)
  unsigned char *img;            // non-NULL: the one-CTA fit packs the tcgen05 operand image of
                                 // searches with n > kDirectMaxN in its tail (score_pack.cuh)
};
// Gram pre-pass on many CTAs (fit.cu): x / l (Xs64) then the kernel matrix tiles (Kt64).
cudaError_t launch_gram(const SearchMeta *meta_d, int S, int nmax, int dmax, const FitIO &io,
                        cudaStream_t stream);
cudaError_t launch_fit(const SearchMeta *meta_d, int S, int smem_bytes, const FitIO &io,
                       SearchMeta *meta_out, cudaStream_t stream, bool pdl);
// Cluster fit (fit_cluster.cu): Cc CTAs per search, the working matrix in their shared memory.
int fit_cluster_smem(int n, int Cc);
bool fit_cluster16_ok(int smem_bytes);
cudaError_t launch_fit_cluster(const SearchMeta *meta_d, int S, int Cc, int smem_bytes,
                               const FitIO &io, SearchMeta *meta_out, cudaStream_t stream);
cudaError_t launch_simt_operands(const SearchMeta *meta_d, int S, const float *X32,
                                 const float *ls32, const double *Linv64, float *Xs32,
                                 float *LT32, cudaStream_t stream);
cudaError_t launch_score_simt(const ScoreLaunch &p, int total_tiles, int dmax, int nmax,
                              cudaStream_t stream);
cudaError_t launch_refine(const RefineLaunch &p, int64_t max_entries, int num_sms, int nmax,
                          cudaStream_t stream);
// O(n^2) append update (append.cu): the previous model's arrays -> the new model's arrays.
struct AppendIO {
  const SearchMeta *prev_meta;   // device meta of the previous model
  const float *prev_X32, *prev_ls32;
  const double *prev_y64, *prev_L64, *prev_Linv64, *prev_Xs64;
  const float *x_new;            // [sum d_s] device
  const double *y_new;           // [S] device
  float *X32, *ls32;
  double *y64, *L64, *Linv64, *Xs64, *alpha64;
};
cudaError_t launch_append(const SearchMeta *meta_in, int S, const AppendIO &io,
                          SearchMeta *meta_out, cudaStream_t stream);
// Precise-mean tier (mean64.cu): float64 mu~ of every row of the precise-tier searches.
// A search is precise when sf2 |alpha|_1 > kMeanTierL1.  SURVEY.md R13 put the float32 mean's
// trouble at |alpha|_1 >~ 1.5e3, but the fast phase's per-candidate bound uses sum_j |k_j alpha_j|,
// which is far smaller for most candidates: measured, the argmax filter stays sparse up to
// |alpha|_1 ~ 3e4 (config 3's searches: 310 .. 2.98e4, ~2.2k refined of 2^24) and collapses for
// BO-like training sets (configs 2/4 in the "bo" layout: |alpha|_1 ~ 1.7e5, every candidate
// flagged).  The tier only changes the cost, never the result (the refine decides every key).
constexpr double kMeanTierL1 = 5.0e4;
cudaError_t launch_mean64(const ScoreLaunch &p, const double *Xs64, int tile, int tile_lo,
                          int tiles, int dmax, double *mean64, const double *etab, int num_sms,
                          cudaStream_t stream);
void mean64_exp_table(double *host);
int mean64_exp_table_size();
// gp_posterior's dense float64 path, candidate-tiled (refine.cu).
cudaError_t launch_posterior64(const RefineLaunch &p, int nmax, int dmax, int num_sms,
                               cudaStream_t stream);
// Small problems: float64 scoring of every row, thread per candidate (refine.cu); n <= 64.
constexpr int kDirectMaxN = 64;
cudaError_t launch_direct(const RefineLaunch &p, int S, int64_t rows, cudaStream_t stream);
}  // namespace gpbo
