/*
 * gpbo.h -- C ABI of libgpbo.so, the B200 (sm_100a) GP-surrogate + Expected-Improvement hot path
 * of arXiv 2403.08131 ("Cost-Effective Methodology for Complex Tuning Searches in HPC").
 *
 * The paper's BO searches (§III.A) train a surrogate on the observed
 * configurations and let "an acquisition function guide the selection of the next
 * configuration"; their cost is "the training complexity of Gaussian Processes ... O(N^3)"
 * (L249, L256, §IV.D).  This library is that step, batched over the many sub-searches the
 * interdependence analysis produces (L163-173, L245-256) and sharded over GPUs:
 *
 *   gp_fit           H1-H4  standardise y, Gram matrix, jittered Cholesky, L^-1, alpha
 *   gp_posterior     H6-H8  posterior mean / latent variance / EI of caller candidates
 *   ei_score_argmax  H6-H10 EI of caller candidates, per-search argmax, cross-GPU max
 *
 * (H* = the step rows of SURVEY.md §8(a); readings R* = SURVEY.md §8(c), listed in DESIGN.md.)
 * The paper names neither kernel nor acquisition (GPTune internals, L77): GP with ARD RBF or
 * Matern-5/2 kernel (reading R1/R2), EI for minimisation with xi = 0
 * (readings R3-R5), ties to the lowest global candidate index.
 *
 * Conventions for every entry point
 *  - Every call returns gpbo_status; no C++ exception crosses the ABI.  On error the message
 *    is available from gpbo_last_error(ctx).
 *  - Calls are ordered on the ctx's CUDA stream and are synchronous on return (they end with
 *    a stream synchronisation because they return host-side results).
 *  - Inputs are read only during the call and remain owned by the caller.  "mem" selects
 *    whether the caller's array pointers are host (GPBO_HOST, any host memory; pinned is
 *    faster) or device (GPBO_DEVICE, on ctx's device) addresses.  Shape arrays (n, d, m_off,
 *    m_global_base) are always host arrays.
 *  - A gpbo_model is library-owned device state until gp_model_free.  A ctx is bound to one
 *    device and stream and is NOT thread-safe.
 *  - Layouts: X and X* are row-major float32 with d_s contiguous encoded coordinates per row,
 *    concatenated over the S searches; y is float64.  Encoded coordinates are expected in
 *    [0, 1] (reading R8) but any finite value is accepted.
 *  - Limits (v1): 1 <= S, 1 <= n_s <= GPBO_MAX_N, 1 <= d_s <= GPBO_MAX_D, M_s < 2^32 - 1.
 *  - Non-finite inputs (X, y, lengthscale, variances) -> GPBO_EINVAL.
 */
#ifndef GPBO_H
#define GPBO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GPBO_MAX_N 512
#define GPBO_MAX_D 64
#define GPBO_NCCL_ID_BYTES 128

typedef enum {
  GPBO_OK = 0,
  GPBO_EINVAL = 1,        /* bad shape / pointer / non-finite input                        */
  GPBO_ENOTPD = 2,        /* Cholesky failed even at the largest jitter (reading R9)       */
  GPBO_WDEGENERATE = 3,   /* warning: constant y; model built with y~ = 0     */
  GPBO_ESAMPLING = 4,     /* candidate generation exhausted (reserved for bo_suggest)     */
  GPBO_ECUDA = 5,         /* CUDA runtime error                                           */
  GPBO_ENCCL = 6,         /* NCCL error                                                   */
  GPBO_ENOMEM = 7,        /* device or pinned host allocation failed                      */
  GPBO_ENOTSUP = 8        /* valid request outside this build's supported envelope        */
} gpbo_status;

typedef enum { GPBO_RBF = 0, GPBO_MATERN52 = 1 } gpbo_kernel;
typedef enum { GPBO_HOST = 0, GPBO_DEVICE = 1 } gpbo_mem;

typedef struct gpbo_ctx gpbo_ctx;
typedef struct gpbo_model gpbo_model;

/* ---------------------------------------------------------------- context
 * gpbo_nccl_unique_id: writes a fresh NCCL unique id (GPBO_NCCL_ID_BYTES bytes) to out; call on
 *   rank 0 and broadcast it (e.g. torch.distributed.broadcast_object_list) to the other ranks.
 * gpbo_ctx_create: binds to CUDA device `device` and stream `cuda_stream` (a cudaStream_t; NULL
 *   = the legacy default stream).  A non-NULL `nccl_unique_id` creates an NCCL communicator of
 *   `nranks` ranks (required when nranks > 1; with nranks == 1 it gives a 1-rank communicator,
 *   so the H10 all-reduce path also runs on one GPU); NULL with nranks == 1 = no communicator.
 *   All ranks must call it collectively.  On success *out owns the communicator and scratch
 *   buffers. */
gpbo_status gpbo_nccl_unique_id(void *out);
gpbo_status gpbo_ctx_create(int device, void *cuda_stream, int nranks, int rank,
                            const void *nccl_unique_id, gpbo_ctx **out);
gpbo_status gpbo_ctx_destroy(gpbo_ctx *ctx);
/* Last error message of this ctx ("" if none).  Valid until the next call on ctx. */
const char *gpbo_last_error(const gpbo_ctx *ctx);
/* Library build string (compile flags, arch) for logs. */
const char *gpbo_version(void);

/* ---------------------------------------------------------------- fit (H1-H4)
 * Ragged batch of S sub-searches.  Search s has n[s] observations of d[s] encoded parameters:
 *   X            float32 [sum n_s d_s]  rows of search s start at sum_{t<s} n_t d_t
 *   y            float64 [sum n_s]      raw objective values, minimised (P L72)
 *   lengthscale  float32 [sum d_s]      ARD lengthscales l > 0 (reading R2: k depends on
 *                                       sum_j ((x_j - x'_j) / l_j)^2)
 *   signal_var   float32 [S]            sf2 > 0, kernel amplitude in standardised units
 *   noise_var    float32 [S]            sn2 >= 0, observation noise in standardised units
 * The fit standardises y (ddof = 0; reading R7), builds K = k(X, X) + (sn2 + j_k) I with the
 * jitter ladder j_k = 1e-8 10^k sf2, k = 0..6 (reading R9), factors K = L L^T in
 * float64 (one CTA per sub-search), forms L^-1 and alpha = K^-1 y~, and stores the scoring
 * operands on the device.  Outputs (host arrays, may be NULL):
 *   status[S]   GPBO_OK | GPBO_ENOTPD | GPBO_WDEGENERATE per search
 *   jitter_k[S] the k that succeeded, -1 on ENOTPD
 * Returns GPBO_ENOTPD if any search failed (the model is still returned; failed searches
 * score no candidate), GPBO_WDEGENERATE if any search is degenerate, else GPBO_OK. */
typedef struct {
  int32_t S;
  const int32_t *n;
  const int32_t *d;
  const float *X;
  const double *y;
  const float *lengthscale;
  const float *signal_var;
  const float *noise_var;
  gpbo_kernel kernel;
  gpbo_mem mem;
} gpbo_fit_args;

gpbo_status gp_fit(gpbo_ctx *ctx, const gpbo_fit_args *args, gpbo_model **out,
                   int32_t *status, int32_t *jitter_k);

/* Asynchronous gp_fit: enqueues the fit on ctx's stream and returns without waiting (GPBO_OK,
 * or GPBO_EINVAL / GPBO_ENOMEM for argument errors detectable on the host).  The per-search
 * statuses stay on the device: scoring calls skip a failed search there (it returns idx -1), and
 * the host copy is refreshed by the next synchronising call (ei_score_argmax, bo_suggest_batch,
 * gp_posterior, gp_model_stats/export) or explicitly by gp_model_sync, which writes status[S] /
 * jitter_k[S] (may be NULL) and returns what gp_fit would have returned (GPBO_EINVAL if an input
 * was non-finite; the model then scores nothing and must still be freed). */
/* Lifetime: with mem = GPBO_DEVICE the fit kernels read the caller's X, y, lengthscale,
 * signal_var and noise_var asynchronously on ctx's stream, so those device buffers must stay
 * valid (not freed, not reused by an allocator on another stream) until ctx's stream has passed
 * the fit -- i.e. until the next synchronising call on ctx returns.  Host inputs (GPBO_HOST) are
 * staged by stream-ordered copies: pageable memory may be reused on return, pinned (page-locked)
 * memory only after the stream has passed the fit.  The Python binding keeps references to the
 * input arrays on the Model until it is freed. */
gpbo_status gp_fit_async(gpbo_ctx *ctx, const gpbo_fit_args *args, gpbo_model **out);
gpbo_status gp_model_sync(gpbo_ctx *ctx, const gpbo_model *model, int32_t *status,
                          int32_t *jitter_k);
void gp_model_free(gpbo_model *model);

/* ---------------------------------------------------------------- append
 * Sequential BO's surrogate update ("re-training the surrogate model"): a new model
 * whose search s holds the previous model's n_s observations plus ONE new one (x_new: d_s
 * encoded values, concatenated over s; y_new[s] raw objective), with the same hyper-parameters
 * and jitter, in O(n^2) per search instead of the O(n^3) refit: the bordered Cholesky
 *   l = L^-1 k(X, x_new),  delta = sqrt(sf2 + sn2 + j - |l|^2),  L' = [L 0; l^T delta],
 *   L'^-1 = [L^-1 0; -(l^T L^-1)/delta 1/delta],
 * then y re-standardised over the n + 1 values (reading R7), alpha = L'^-T L'^-1 y~ and the
 * diagnostics / LML recomputed.  Equal to a full gp_fit of the n + 1 observations up to float64
 * rounding (Cholesky is unique and the full fit's jitter ladder stops at the same k).  If the
 * bordered matrix is not positive definite at the old jitter (delta^2 <= 0) the whole batch is
 * refitted from scratch with the jitter ladder (gpbo_last_append_refit(ctx) = 1).  x_new / y_new
 * are host or device arrays per `mem`; `prev` is left unchanged (free it when done).  Outputs and
 * return codes as gp_fit; GPBO_EINVAL if a previous search has no fit, n_s + 1 > 512 or a new
 * value is non-finite.  Synchronous. */
gpbo_status gp_fit_append(gpbo_ctx *ctx, const gpbo_model *prev, const float *x_new,
                          const double *y_new, gpbo_mem mem, gpbo_model **out, int32_t *status,
                          int32_t *jitter_k);
int64_t gpbo_last_append_refit(const gpbo_ctx *ctx);

/* Log marginal likelihood of every search's fit (host array lml[S], standardised targets):
 *   log p(y~ | X, theta) = -1/2 y~^T alpha - sum_i log L_ii - n/2 log(2 pi)
 * with K = k(X, X) + (sn2 + j_k) I the (jittered) matrix actually factored (Rasmussen & Williams
 * eq. 2.30; the GP "training" whose O(N^3) cost PAPER.md L249 names).  -inf for failed fits. */
gpbo_status gp_model_lml(const gpbo_model *model, double *lml);

/* ---------------------------------------------------------------- ML-II
 * Hyper-parameters by maximising the log marginal likelihood (type-II maximum likelihood), per
 * search, with multi-start Nelder-Mead in log space (8 seeded starts, 200
 * iterations each; bounds lengthscale [1e-3, 10], signal [1e-3, 1e3], noise [1e-6, 1] in
 * standardised units).  theta = (log l_1 .. log l_d, log sf2, log sn2); start 0 is the theta in
 * `args`, starts 1.. are uniform in the log box from a counter-based generator (splitmix64, see
 * ml2.cuh); simplex step `step` (log units); reflection 1, expansion 2, contraction 1/2, shrink
 * 1/2; points clamped to the box; exactly `iters` iterations.  All (search, start) simplices
 * advance together: each round evaluates every requested point as ONE batched gp_fit launch
 * (fit.cu, one CTA per point).  Inputs: `args` with mem = GPBO_HOST (its lengthscale /
 * signal_var / noise_var = start 0).  Outputs (host): the best theta per search (ls_out [sum d],
 * sf2_out [S], sn2_out [S], as float32 exactly as evaluated), its LML (lml_out [S], may be NULL)
 * and the LML of every start point (lml_starts [S * starts], may be NULL).  Invariant:
 * lml_out[s] >= lml_starts[s * starts + k] for every k.  Refit with gp_fit to score. */
typedef struct {
  int32_t starts;   /* multi-start count (SPEC: 8)                                        */
  int32_t iters;    /* Nelder-Mead iterations per start (SPEC: 200)                       */
  uint64_t seed;    /* start-point generator seed                                         */
  double step;      /* initial simplex step in log units (0.5)                            */
  double ls_lo, ls_hi, sf2_lo, sf2_hi, sn2_lo, sn2_hi;  /* bounds (SPEC L376 above)        */
} gpbo_ml2_opts;
gpbo_status gp_fit_ml2(gpbo_ctx *ctx, const gpbo_fit_args *args, const gpbo_ml2_opts *opts,
                       float *ls_out, float *sf2_out, float *sn2_out, double *lml_out,
                       double *lml_starts);
/* LML evaluations (batched fit searches) the last gp_fit_ml2 call on ctx ran. */
int64_t gpbo_last_ml2_evals(const gpbo_ctx *ctx);

/* Fitted per-search statistics (host copies, any may be NULL): y mean and std (raw units),
 * best = min y~ (standardised), alpha_l1 = ||alpha||_1 (the mu-tier diagnostic, reading R13). */
gpbo_status gp_model_stats(const gpbo_model *model, int32_t s, double *mean, double *std,
                           double *best, double *alpha_l1);

/* Test/diagnostic export of the float64 fit of search s into caller host buffers of n_s*n_s
 * (L, Linv: row-major, lower triangle, upper zero) and n_s (alpha) doubles; any may be NULL. */
gpbo_status gp_model_export(gpbo_ctx *ctx, const gpbo_model *model, int32_t s, double *L,
                            double *Linv, double *alpha);

/* ---------------------------------------------------------------- posterior (H6-H8, H11)
 * Scores M candidates X* (float32 [M d_s], row-major) of search s and writes, per candidate,
 *   mu  = mean + std mu~       (raw units; mu~ = k*^T alpha)
 *   var = std^2 s2~            (latent variance, raw units^2; s2~ = max(sf2 - |L^-1 k*|^2, 0))
 *   ei  = std EI(mu~, s2~, best)  (raw units; best = min y~)
 * to float32 arrays in `mem` space (any may be NULL).  Same kernel as ei_score_argmax. */
gpbo_status gp_posterior(gpbo_ctx *ctx, const gpbo_model *model, int32_t s, const float *Xstar,
                         int64_t M, gpbo_mem mem, float *mu, float *var, float *ei);

/* ---------------------------------------------------------------- EI + argmax (H6-H10)
 * Scores this rank's shard of every search's candidate pool and returns the global argmax.
 *   Xstar          float32, concatenation over s of this rank's rows of search s (M_s_local x d_s)
 *   m_off          int64 [S+1] host: rows of search s are Xstar rows [m_off[s], m_off[s+1])
 *   m_global_base  int64 [S] host: global candidate index of this rank's first row of search s
 *                  (NULL = 0); ties resolve to the lowest GLOBAL index (reading R10)
 *   best           float64 [S] host: incumbent in raw units (NULL = min observed y; R3)
 * Outputs (host, any may be NULL):
 *   idx[S]  global index of the suggestion, -1 if search s had no scorable candidate
 *   ei[S]   its EI in raw units (std * EI~)
 * With nranks > 1 every rank returns the same result: the per-search 64-bit keys
 * (EI~ bits << 32 | (2^32 - 1 - idx)) are combined with one ncclAllReduce(max) on ctx's
 * communicator (H10). */
gpbo_status ei_score_argmax(gpbo_ctx *ctx, const gpbo_model *model, const float *Xstar,
                            const int64_t *m_off, const int64_t *m_global_base,
                            const double *best, gpbo_mem mem, int64_t *idx, float *ei);

/* ---------------------------------------------------------------- spaces and suggestions
 * (H0 encoding, H5 candidate generation, bo_suggest_batch)
 * A search space (Table IV, constraints L391): P parameters in
 * declaration order, each
 *   GPBO_P_REAL        [lo, hi)            encoded (v - lo)/(hi - lo)
 *   GPBO_P_INT         lo..hi (step 1)     encoded (v - lo)/(hi - lo)
 *   GPBO_P_ORDINAL     K numeric values    encoded rank/(K-1) (K = 1 -> 0)
 *   GPBO_P_CATEGORICAL K labels 0..K-1     encoded one-hot (K columns)
 *   GPBO_P_FIXED       the value lo        no encoded column, draws nothing (a parameter the
 *                                          interdependence plan does not tune in this search:
 *                                          fixed at its default / an earlier stage's value;
 *                                          SPEC.md L243, L290) -- decoded as lo
 * (reading R8), plus constrained blocks: a block names >= 1 discrete parameters and lists its
 * valid value-index tuples; the generator draws one tuple uniformly (no rejection), so every
 * candidate satisfies the caller's constraints.  Encoded dimension d = number of
 * non-fixed, non-categorical parameters + sum of categorical K (<= GPBO_MAX_D).
 * Generator: Philox4x32-10, key = seed, word u of global candidate i of search s at iteration t
 * = output[u % 4] of Philox(ctr = (i, s, t, u / 4)), u over free parameters (declaration order)
 * then blocks; real: (w >> 8) 2^-24, K values: (u64(w >> 8) K) >> 24. */
typedef enum { GPBO_P_REAL = 0, GPBO_P_INT = 1, GPBO_P_ORDINAL = 2, GPBO_P_CATEGORICAL = 3,
               GPBO_P_FIXED = 4 }
    gpbo_param_kind;
typedef struct gpbo_space gpbo_space;
typedef struct {
  int32_t P;
  const int32_t *kind;        /* [P] gpbo_param_kind                                          */
  const int32_t *nvals;       /* [P] K for ORDINAL / CATEGORICAL (ignored otherwise)          */
  const double *lo, *hi;      /* [P] range for REAL / INT (ignored otherwise)                 */
  const int32_t *val_off;     /* [P] offset of the ORDINAL value list in values (may be NULL  */
  const double *values;       /*     when there is no ORDINAL parameter)                      */
  int32_t nblocks;
  const int32_t *block_off;   /* [nblocks+1] offsets into block_params                        */
  const int32_t *block_params;/* parameter indices; each discrete, in at most one block       */
  const int32_t *tuple_off;   /* [nblocks+1] offsets in tuples (counted in tuples)            */
  const int32_t *tuples;      /* block b: tuple_off[b+1]-tuple_off[b] tuples of block-size     */
} gpbo_space_desc;            /* value indices, blocks concatenated                            */

/* All host arrays; copied (the space is immutable).  GPBO_ESAMPLING if a block has no valid
 * tuple (an unsatisfiable constraint). */
gpbo_status gpbo_space_create(gpbo_ctx *ctx, const gpbo_space_desc *desc, gpbo_space **out);
void gpbo_space_free(gpbo_space *space);
int32_t gpbo_space_dim(const gpbo_space *space);
/* Host helper (H0): encode one raw configuration raw[P] -> enc[d] exactly as the generator does
 * (callers encode their observation history with it).  GPBO_EINVAL for out-of-domain values. */
gpbo_status gpbo_space_encode(const gpbo_space *space, const double *raw, float *enc);
/* H5 alone (tests): encoded candidates first_idx .. first_idx+count-1 of (seed, search,
 * iteration) -> enc[count * d] float32 in `mem` space. */
gpbo_status gpbo_space_sample(gpbo_ctx *ctx, const gpbo_space *space, uint64_t seed,
                              int32_t search, int32_t iteration, int64_t first_idx,
                              int64_t count, gpbo_mem mem, float *enc);
/* One BO suggestion per sub-search (the acquisition step of P:L72): for every search s, draw the
 * M[s] candidates of (seed, s, iteration) on the device (this rank scores its contiguous shard
 * of each pool, global indices as in ei_score_argmax), optionally mask candidates equal to an
 * observed configuration of the model (dedup != 0, reading R14), score them (H6-H9, float64
 * refine), combine across ranks (H10) and decode the winner (H11).  Outputs (host):
 *   idx[S]     global candidate index (-1 if none), identical on every rank
 *   x_raw[sum P_s]  the winner's raw parameter values (concatenated per search; REAL exact to
 *              float64, others the chosen value / label index)
 *   ei[S]      its EI in raw units
 * spaces[s] must have dimension d_s of the model. */
gpbo_status bo_suggest_batch(gpbo_ctx *ctx, const gpbo_model *model,
                             const gpbo_space *const *spaces, const int64_t *M, uint64_t seed,
                             int32_t iteration, int32_t dedup, int64_t *idx, double *x_raw,
                             float *ei);

/* ---------------------------------------------------------------- planner
 * Host-only (no GPU needed): the methodology's interdependence analysis, which emits the batch of
 * sub-searches the calls above fit and score (§IV.B-D, §VIII).
 *
 * gpbo_influence (§IV.B): matrix[r * P + p] = (1/V') sum_i |(baseline[r] - t_i) /
 *   baseline[r]| over the valid variations i of parameter p (valid [P * V] may be NULL = all;
 *   V' = their count; NaN when none is valid -- "unknown", not 0), t_i = variations[(p * V + i) *
 *   R + r] (routine r's runtime with parameter p at its i-th variation, all others at baseline).
 *   GPBO_EINVAL for a zero or non-finite baseline.
 * gpbo_plan: routines r (parent[r] = enclosing region or -1; has_metric[r] = its own runtime is
 *   measured) own parameters (owners[owner_off[p] .. owner_off[p+1]): >= 1 routine; several =
 *   one kernel used in several regions); shared[p] = 1 when p must keep one value across the
 *   application.  Routines with a metric and no children are the stage-2 candidates; the others
 *   (outer regions, routines without a metric such as the MPI grid) get stage-1 searches against
 *   their metric or the total objective (target -1).  Steps (deterministic, ties -> lower index):
 *   shared kernels -> owner of highest influence (step 5, L545); a child parameter above the
 *   cut-off on its parent and on >= 2 sibling children moves to the parent's search (L543);
 *   cross edges >= cutoff (L235, L254) merge the two routines (shared[p]; union-find) or
 *   duplicate p into the target's search ("tune twice", L237); a search above dim_cap keeps its
 *   dim_cap most influential parameters (max over its routines; L167, L249) and drops the rest
 *   to defaults; budget = max(budget_floor, budget_mult * dims) (L256).
 *   Outputs (caller arrays sized for R searches): nsearch; per search s: stage (1, 2), target
 *   routine (-1 = total), budget, dims; tuned[s * P + p] = 1 if s tunes p; dropped[p] = 1 if no
 *   search tunes p (fixed at its default). */
typedef struct {
  int32_t R, P;
  const int32_t *parent;      /* [R] */
  const int32_t *has_metric;  /* [R] */
  const int32_t *owner_off;   /* [P + 1] */
  const int32_t *owners;      /* [owner_off[P]] */
  const int32_t *shared;      /* [P] */
  const double *matrix;       /* [R * P] variability (fractions; 1.0 = 100 %) */
  double cutoff;              /* e.g. 0.25 synthetic (L254), 0.10 RT-TDDFT (L543) */
  int32_t dim_cap;            /* 10 (L167) */
  int32_t budget_mult, budget_floor;  /* 10, 10 (L256 "at least 10 x num_parameters") */
} gpbo_plan_args;
typedef struct {
  int32_t nsearch;
  int32_t *search_stage, *search_target, *search_budget, *search_dims;  /* [R] */
  uint8_t *tuned;    /* [R * P] */
  uint8_t *dropped;  /* [P] */
} gpbo_plan_out;
gpbo_status gpbo_influence(int32_t R, int32_t P, int32_t V, const double *baseline,
                           const double *variations, const uint8_t *valid, double *matrix);
gpbo_status gpbo_plan(const gpbo_plan_args *args, gpbo_plan_out *out);

/* Number of CUDA kernels the library launched on ctx since creation (for bench accounting). */
int64_t gpbo_launch_count(const gpbo_ctx *ctx);

/* ncclAllReduce calls (H10) ctx has issued on its communicator since creation. */
int64_t gpbo_collective_count(const gpbo_ctx *ctx);

/* Soundness check of the last argmax call (ei_score_argmax / bo_suggest_batch): the number of
 * refined or audited candidates whose float64 EI fell outside the fast phase's EI bracket.  A
 * search with any violation was re-scored exactly (every row in float64) before its result was
 * decoded, so a failed error bound costs time, never a wrong suggestion.  Expected: 0. */
int64_t gpbo_last_bracket_violations(const gpbo_ctx *ctx);


/* Candidates the last ei_score_argmax call on ctx re-scored in the float64 refine phase
 * (those whose fast-phase EI upper bound reached the running per-search maximum lower bound). */
int64_t gpbo_last_refine_count(const gpbo_ctx *ctx);
/* Fast-phase implementation of the last scoring call: 1 = CUDA-core, 2 = tcgen05 with the
 * shared-memory-resident operand image, 3 = tcgen05 with streamed operands, 4 = float64 direct
 * (small problems; no refine phase), 5 = float64 dense refine of every row (gp_posterior beyond
 * the direct kernel's envelope: no fast phase). */
int gpbo_last_score_impl(const gpbo_ctx *ctx);
/* 1 if the last scoring call's tcgen05 fast phase (impl 2) ran as CTA pairs (cta_group::2,
 * M = 256 MMAs over two SMs; chosen for models whose searches all have n > 112 and whose pair
 * image fits; GPBO_TC_PAIR=0 in the environment disables it), else 0. */
int gpbo_last_tc_pair(const gpbo_ctx *ctx);

/* Per-kernel timing with CUDA events recorded on ctx's stream around every library kernel
 * launch (for bench.py's roofline).  gpbo_set_profiling(ctx, 1) enables it and clears the
 * totals; gpbo_kernel_time returns the launch count and summed milliseconds of one kind:
 * 0 = fit (H1-H4), 1 = scoring fast phase (H6-H9), 2 = float64 refine phase, 3 = operand pack,
 * 4 = precise-mean tier (float64 mu~ for searches with sf2 |alpha|_1 > 5e4, reading R13). */
gpbo_status gpbo_set_profiling(gpbo_ctx *ctx, int on);
gpbo_status gpbo_kernel_time(gpbo_ctx *ctx, int kind, int64_t *count, double *ms);





/* Test and diagnostic hooks (implementation forcing, error-bound scaling, pipeline traces,
 * microbenchmarks, the host Nelder-Mead self-test) are declared in gpbo_test.h. */

#ifdef __cplusplus
}
#endif
#endif /* GPBO_H */
