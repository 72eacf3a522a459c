// Host side of the C ABI declared in include/gpbo.h: argument validation, model/ctx lifecycle,
// stream-ordered staging of host inputs, kernel launches and the NCCL max-all-reduce of the
// per-search argmax keys (H10).  No numerical work happens here: every step of the path runs in
// the CUDA kernels of fit.cu / score_*.cu.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gpbo_internal.cuh"
#include "ml2.cuh"
#include "score_tc.cuh"
#include "space_internal.cuh"

using gpbo::SearchMeta;

struct gpbo_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int nranks = 1, rank = 0;
  ncclComm_t comm = nullptr;
  std::string err;
  unsigned long long *keys_d = nullptr;  // [cap] keys | [cap] u32 thresholds | u32 list count
  unsigned long long *keys_h = nullptr;
  int keys_cap = 0;
  unsigned long long *cur_keys_d = nullptr;  // this call's keys | viol | thr | count (in aux_d)
  size_t cur_key_bytes = 0;
  const int64_t *cur_p_off = nullptr;  // this call's device m_off | m_base | x_off | best (aux_d)
  int64_t last_violations = 0;  // bracket violations found by the last argmax call
  int64_t last_ml2_evals = 0;   // LML evaluations of the last gp_fit_ml2 call
  int64_t last_append_refit = 0;  // the last gp_fit_append fell back to a full refit
  float bound_scale = 1.f;      // error-bound multiplier of the fast phase (test hook)
  gpbo::RefineEntry *list_d = nullptr;   // refine list of the argmax path
  size_t list_cap = 0;
  void *stage_d = nullptr;  // device staging of host-resident candidates / outputs
  size_t stage_cap = 0;
  void *aux_d = nullptr;    // per-call small arrays (offsets, bases, best, tile prefix)
  void *aux_h = nullptr;    // pinned mirror
  void *meta_h = nullptr;   // pinned staging of the fit's meta records
  size_t meta_cap = 0;
  cudaEvent_t meta_ev = nullptr;  // recorded after the upload that reads meta_h
  cudaEvent_t aux_ev = nullptr;   // recorded after the upload that reads aux_h
  size_t aux_cap = 0;
  int64_t launches = 0;
  int64_t collectives = 0;  // ncclAllReduce calls issued on comm
  // optional per-kernel CUDA-event timing (gpbo_set_profiling): kinds fit / fast / refine / pack
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_open;
  double kern_ms[5] = {0, 0, 0, 0, 0};
  int64_t kern_count[5] = {0, 0, 0, 0, 0};
  double *mean_d = nullptr;  // precise-tier float64 means of the current scoring call
  size_t mean_cap = 0;
  double *etab_d = nullptr;  // e^{-k/16} table of the precise tier
  int64_t last_refine = 0;
  int last_impl = 0;
  int last_pair = 0;  // the last tcgen05 fast phase ran as CTA pairs
  unsigned long long *trace = nullptr;  // device buffer for the next tcgen05 launch        // 1 = CUDA-core, 2 = tcgen05 fast phase in the last scoring call  // candidates the last argmax call flagged for the refine phase
  int num_sms = 148;
  // chunked host feed of ei_score_argmax (mem = GPBO_HOST): candidate chunks are copied on
  // copy_stream while the tcgen05 kernel scores the previous chunk on `stream`
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t feed_ev[8] = {};
  // bo_suggest_batch draws its candidates on gen_stream, overlapping a pending fit on `stream`:
  // xready_ev marks the latest Gram pre-pass (which copies X into the model, the dedup's input)
  cudaStream_t gen_stream = nullptr;
  cudaEvent_t gen_ev = nullptr, xready_ev = nullptr;
  int score_impl = 0;       // 0 = auto (tcgen05 where supported), 1 = SIMT, 2 = tcgen05,
                            // 3 = tcgen05 with the streamed image layout forced at fit time,
                            // 4 = float64 direct kernel (n <= 64)
};

struct gpbo_model {
  int S = 0;
  int kernel = 0;
  int device = 0;
  int nmax = 0, dmax = 0;
  cudaStream_t stream = nullptr;
  std::vector<SearchMeta> meta;  // host copy (after the fit)
  SearchMeta *meta_d = nullptr;
  char *block = nullptr;         // one cudaMallocAsync block, sub-allocated below
  float *X32 = nullptr, *ls32 = nullptr, *Xs32 = nullptr, *LT32 = nullptr;
  double *y64 = nullptr, *L64 = nullptr, *Linv64 = nullptr, *alpha64 = nullptr;
  double *Xs64 = nullptr;
  unsigned char *img = nullptr;  // tcgen05 operand images
  int64_t img_bytes = 0;
  mutable bool simt_ready = false;  // Xs32 / LT32 built (on first CUDA-core scoring call)
  mutable bool packed = false;      // tcgen05 operand images built (on first tcgen05 call)
  mutable bool meta_pending = false;  // gp_fit_async: host meta not yet refreshed from the device
  int64_t nx_total = 0, nls_total = 0, ny_total = 0;  // sum n d, sum d, sum n
};

namespace {

gpbo_status fail(gpbo_ctx *ctx, gpbo_status st, const std::string &msg) {
  if (ctx) ctx->err = msg;
  return st;
}

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? GPBO_ENOMEM : GPBO_ECUDA,    \
                  std::string(#x) + ": " + cudaGetErrorString(e_));                   \
  } while (0)

#define NK(x)                                                                         \
  do {                                                                                \
    ncclResult_t r_ = (x);                                                            \
    if (r_ != ncclSuccess)                                                            \
      return fail(ctx, GPBO_ENCCL, std::string(#x) + ": " + ncclGetErrorString(r_));  \
  } while (0)

inline int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

enum { kKernFit = 0, kKernFast = 1, kKernRefine = 2, kKernPack = 3, kKernMean = 4 };

cudaEvent_t take_event(gpbo_ctx *ctx) {
  if (!ctx->ev_pool.empty()) {
    cudaEvent_t e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Brackets one library kernel launch with events on ctx's stream when profiling is on.
struct KernTimer {
  gpbo_ctx *ctx;
  int kind;
  cudaEvent_t a = nullptr, b = nullptr;
  KernTimer(gpbo_ctx *c, int k) : ctx(c), kind(k) {
    if (!ctx->profiling) return;
    a = take_event(ctx);
    b = take_event(ctx);
    cudaEventRecord(a, ctx->stream);
  }
  ~KernTimer() {
    if (!a) return;
    cudaEventRecord(b, ctx->stream);
    ctx->ev_open.push_back({kind, {a, b}});
  }
};

// Called after a stream synchronisation: fold the closed event pairs into the totals.
void harvest_events(gpbo_ctx *ctx) {
  for (auto &o : ctx->ev_open) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, o.second.first, o.second.second) == cudaSuccess) {
      ctx->kern_ms[o.first] += ms;
      ctx->kern_count[o.first] += 1;
    }
    ctx->ev_pool.push_back(o.second.first);
    ctx->ev_pool.push_back(o.second.second);
  }
  ctx->ev_open.clear();
}

gpbo_status ensure_stage(gpbo_ctx *ctx, size_t bytes) {
  if (bytes <= ctx->stage_cap) return GPBO_OK;
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->stage_d) CK(cudaFree(ctx->stage_d));
  ctx->stage_d = nullptr;
  ctx->stage_cap = 0;
  CK(cudaMalloc(&ctx->stage_d, bytes));
  ctx->stage_cap = bytes;
  return GPBO_OK;
}

gpbo_status ensure_mean(gpbo_ctx *ctx, size_t rows) {
  if (!ctx->etab_d) {  // the precise tier's e^{-k/16} table (mean64.cu), once per ctx
    std::vector<double> t(gpbo::mean64_exp_table_size());
    gpbo::mean64_exp_table(t.data());
    CK(cudaMalloc(&ctx->etab_d, t.size() * sizeof(double)));
    CK(cudaMemcpy(ctx->etab_d, t.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  if (rows <= ctx->mean_cap) return GPBO_OK;
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->mean_d) CK(cudaFree(ctx->mean_d));
  ctx->mean_d = nullptr;
  ctx->mean_cap = 0;
  const size_t cap = std::max<size_t>(rows, 1 << 16);
  CK(cudaMalloc(&ctx->mean_d, cap * sizeof(double)));
  ctx->mean_cap = cap;
  return GPBO_OK;
}

gpbo_status ensure_aux(gpbo_ctx *ctx, size_t bytes) {
  if (bytes <= ctx->aux_cap) return GPBO_OK;
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->aux_d) CK(cudaFree(ctx->aux_d));
  if (ctx->aux_h) CK(cudaFreeHost(ctx->aux_h));
  ctx->aux_d = ctx->aux_h = nullptr;
  size_t cap = std::max<size_t>(bytes, 1 << 16);
  CK(cudaMalloc(&ctx->aux_d, cap));
  CK(cudaMallocHost(&ctx->aux_h, cap));
  ctx->aux_cap = cap;
  return GPBO_OK;
}

gpbo_status ensure_meta_h(gpbo_ctx *ctx, size_t bytes) {
  if (bytes <= ctx->meta_cap) return GPBO_OK;
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->meta_h) CK(cudaFreeHost(ctx->meta_h));
  ctx->meta_h = nullptr;
  const size_t cap = std::max<size_t>(bytes, 1 << 14);
  CK(cudaMallocHost(&ctx->meta_h, cap));
  ctx->meta_cap = cap;
  return GPBO_OK;
}

// Host copy of the fit results of an asynchronously fitted model (blocking; not on the hot path
// of the scoring call, which refreshes it in its own final synchronisation).
gpbo_status refresh_meta(const gpbo_model *model) {
  if (!model->meta_pending) return GPBO_OK;
  gpbo_model *m = const_cast<gpbo_model *>(model);
  if (cudaMemcpyAsync(m->meta.data(), m->meta_d, sizeof(SearchMeta) * m->S,
                      cudaMemcpyDeviceToHost, m->stream) != cudaSuccess ||
      cudaStreamSynchronize(m->stream) != cudaSuccess)
    return GPBO_ECUDA;
  m->meta_pending = false;
  return GPBO_OK;
}

gpbo_status ensure_keys(gpbo_ctx *ctx, int S) {
  if (S <= ctx->keys_cap) return GPBO_OK;
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->keys_d) CK(cudaFree(ctx->keys_d));
  if (ctx->keys_h) CK(cudaFreeHost(ctx->keys_h));
  int cap = std::max(S, 64);
  CK(cudaMalloc(&ctx->keys_d, cap * (sizeof(unsigned long long) + 4) + 16));
  CK(cudaMallocHost(&ctx->keys_h, (3 * cap + 2) * sizeof(unsigned long long)));
  ctx->keys_cap = cap;
  return GPBO_OK;
}

gpbo_status ensure_list(gpbo_ctx *ctx, size_t entries) {
  if (entries <= ctx->list_cap) return GPBO_OK;
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->list_d) CK(cudaFree(ctx->list_d));
  ctx->list_d = nullptr;
  ctx->list_cap = 0;
  size_t cap = std::max<size_t>(entries, 1 << 16);
  CK(cudaMalloc(&ctx->list_d, cap * sizeof(gpbo::RefineEntry)));
  ctx->list_cap = cap;
  return GPBO_OK;
}

struct Outputs {
  float *mu = nullptr, *var = nullptr, *ei = nullptr;   // posterior mode (device)
  float *dbg[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // debug mode
};

// Shared scoring launch used by gp_posterior and ei_score_argmax: the fast phase (tcgen05 or
// CUDA-core kernel) followed by the float64 refine phase.
// host_src (optional): the caller's host copy of the candidates; Xstar_dev is then the device
// staging buffer they are copied into, here -- in chunks overlapped with the scoring of the
// previous chunk when the tcgen05 kernels run, else in one copy.
gpbo_status run_score(gpbo_ctx *ctx, const gpbo_model *model, int s_first, int S,
                      const float *Xstar_dev, const int64_t *m_off, const int64_t *m_base,
                      const double *best_std, int mode, const Outputs &out,
                      const float *host_src = nullptr) {
  // aux layout: m_off[S+1] i64 | m_base[S] i64 | x_off[S] i64 | best[S] f64 | tile_first[S+1] i32
  // | (8-aligned) keys[S] u64 | viol[S] u64 | thr[S] u32 | list count u32 -- the key /
  // violation / threshold / count words are zeroed by the same upload (no separate memset) and
  // read back by one copy; keys and viol are adjacent so one all-reduce(max) covers both
  const size_t meta_bytes = ((size_t)(S + 1) * 8 + (size_t)S * 24 + (size_t)(S + 1) * 4 + 7) & ~(size_t)7;
  const size_t key_bytes = (size_t)S * 20 + 4;
  const size_t bytes = meta_bytes + key_bytes;
  gpbo_status st = ensure_aux(ctx, bytes + 64);
  if (st) return st;
  st = ensure_keys(ctx, S);
  if (st) return st;
  if (ctx->aux_ev) CK(cudaEventSynchronize(ctx->aux_ev));  // aux_h may feed an earlier copy
  char *h = (char *)ctx->aux_h;
  int64_t *h_off = (int64_t *)h;
  int64_t *h_base = h_off + (S + 1);
  int64_t *h_xoff = h_base + S;
  double *h_best = (double *)(h_xoff + S);
  int32_t *h_tiles = (int32_t *)(h_best + S);
  // pick the implementation: tcgen05 when every search fits its envelope
  bool use_tc = ctx->score_impl != 1 && ctx->score_impl != 4;
  bool use_tcs = use_tc;  // the streamed tcgen05 kernel
  int nmax = 0, dmax = 0;
  double work = 0.0;  // sum over searches of rows x n16^2 (the direct kernel's cost)
  for (int i = 0; i < S; ++i) {
    const SearchMeta &m = model->meta[s_first + i];
    nmax = std::max(nmax, m.n);
    dmax = std::max(dmax, m.d_pad);
    if (!gpbo::tc_supported(m)) use_tc = false;
    if (!gpbo::tcs_supported(m)) use_tcs = false;
    const double n16 = (double)((m.n + 15) & ~15);
    work += (double)(m_off[i + 1] - m_off[i]) * n16 * n16;
  }
  if (use_tcs) use_tc = true;
  // small problems (config 1, the first BO iterations): one float64 kernel scores every row
  // exactly -- no operand image, no fast phase, no refine (auto below 2^24 row x n16^2, or
  // forced by impl 4); n <= 64 only
  const bool direct = mode != gpbo::kModeDebug && nmax <= gpbo::kDirectMaxN &&
                      (ctx->score_impl == 4 || (ctx->score_impl == 0 && work <= 16777216.0));
  if (direct) use_tc = use_tcs = false;
  // gp_posterior outside the direct kernel's envelope: every row is scored by the float64 dense
  // refine (its mu / var / EI outputs); the fast phase would only be recomputed there, so it is
  // not launched (nor the operand pack)
  const bool dense_only = mode == gpbo::kModePosterior && !direct;
  if (dense_only) use_tc = use_tcs = false;
  if (ctx->score_impl == 2 && !use_tc && !dense_only)
    return fail(ctx, GPBO_ENOTSUP, "tcgen05 scoring requested outside its supported envelope");
  const int tile = use_tc ? gpbo::kTcTile : gpbo::kSimtTile;  // (direct: any)
  // CTA-pair kernel: every search gets an even tile count (whole 256-row pair tiles; the second
  // half of a ragged pair tile scores nothing)
  const bool pair = use_tc && !use_tcs && model->meta[s_first].tc_pair;
  h_tiles[0] = 0;
  int64_t xo = 0;
  for (int i = 0; i < S; ++i) {
    h_xoff[i] = xo;
    xo += (m_off[i + 1] - m_off[i]) * model->meta[s_first + i].d;
    h_off[i] = m_off[i] - m_off[0];
    h_base[i] = m_base ? m_base[i] : 0;
    h_best[i] = best_std[i];
    const int64_t Ms = m_off[i + 1] - m_off[i];
    if (Ms < 0 || h_base[i] < 0 || h_base[i] + Ms >= 0xFFFFFFFFll)
      return fail(ctx, GPBO_EINVAL, "candidate offsets out of range (M_s must be < 2^32-1)");
    const int st_i = model->meta[s_first + i].status;
    // an asynchronous fit's status is not known here: its tiles run and the kernels skip a
    // failed search on the device
    const bool fitted = model->meta_pending || st_i == GPBO_OK || st_i == GPBO_WDEGENERATE;
    int64_t t = fitted ? (Ms + tile - 1) / tile : 0;  // failed fits score nothing
    if (pair) t = (t + 1) & ~(int64_t)1;
    if ((int64_t)h_tiles[i] + t > (1ll << 30))
      return fail(ctx, GPBO_EINVAL, "too many candidates in one call");
    h_tiles[i + 1] = h_tiles[i] + (int32_t)t;
  }
  h_off[S] = m_off[S] - m_off[0];
  const int64_t rows = h_off[S];
  if (mode == gpbo::kModeArgmax) {
    st = ensure_list(ctx, (size_t)rows);
    if (st) return st;
  }
  std::memset((char *)ctx->aux_h + meta_bytes, 0, key_bytes);
  CK(cudaMemcpyAsync(ctx->aux_d, ctx->aux_h, bytes, cudaMemcpyHostToDevice, ctx->stream));
  if (!ctx->aux_ev) CK(cudaEventCreateWithFlags(&ctx->aux_ev, cudaEventDisableTiming));
  CK(cudaEventRecord(ctx->aux_ev, ctx->stream));
  // operand preparation after the upload, so the scoring kernel directly follows the pack on the
  // stream: its programmatic dependent launch overlaps barrier init / TMEM allocation with it
  if (use_tc && !model->packed) {
    KernTimer t(ctx, kKernPack);
    CK(gpbo::launch_pack_tc(model->meta_d, model->S, model->Linv64, model->Xs64, model->alpha64,
                            model->ls32, model->img, ctx->stream));
    ctx->launches += 1;
    model->packed = true;
  }
  if (!use_tc && !direct && !dense_only && !model->simt_ready) {
    CK(gpbo::launch_simt_operands(model->meta_d, model->S, model->X32, model->ls32,
                                  model->Linv64, model->Xs32, model->LT32, ctx->stream));
    ctx->launches += 1;
    model->simt_ready = true;
  }
  unsigned long long *keys_d = (unsigned long long *)((char *)ctx->aux_d + meta_bytes);
  unsigned long long *viol_d = keys_d + S;
  unsigned int *thr_d = (unsigned int *)(keys_d + 2 * S);
  unsigned int *count_d = thr_d + S;
  ctx->cur_keys_d = keys_d;
  ctx->cur_key_bytes = key_bytes;
  ctx->cur_p_off = (const int64_t *)ctx->aux_d;
  char *dptr = (char *)ctx->aux_d;
  gpbo::ScoreLaunch p{};
  p.meta = model->meta_d + s_first;
  p.Xstar = Xstar_dev;
  p.m_off = (const int64_t *)dptr;
  p.m_base = p.m_off + (S + 1);
  p.x_off = p.m_base + S;
  p.best = (const double *)(p.x_off + S);
  p.tile_first = (const int32_t *)(p.best + S);
  p.S = S;
  p.Xs32 = model->Xs32;
  p.LT32 = model->LT32;
  p.alpha64 = model->alpha64;
  p.ls32 = model->ls32;
  p.img = model->img;
  p.keys = keys_d;
  p.out_var = out.var;
  p.mode = mode;
  p.thr = thr_d;
  p.list = ctx->list_d;
  p.list_count = count_d;
  p.list_cap = (uint32_t)std::min<size_t>(ctx->list_cap, 0xFFFFFFFFu);
  p.dbg_mu = out.dbg[0]; p.dbg_dmu = out.dbg[1]; p.dbg_var = out.dbg[2];
  p.dbg_dvar = out.dbg[3]; p.dbg_eilo = out.dbg[4]; p.dbg_eihi = out.dbg[5];
  p.trace = ctx->trace;
  p.bound_scale = ctx->bound_scale >= 0.f ? ctx->bound_scale : 1.f;
  p.break_bracket = ctx->bound_scale < 0.f ? 1 : 0;
  const int tiles = h_tiles[S];
  ctx->last_impl = direct ? 4 : dense_only ? 5 : use_tcs ? 3 : use_tc ? 2 : 1;
  ctx->last_pair = pair && !direct && !dense_only ? 1 : 0;
  const int64_t floats_all = xo;
  // element offset in X* of the first row of tile t (tile indices of this call)
  auto tile_elem = [&](int t) -> int64_t {
    if (t >= tiles) return floats_all;
    int i = (int)(std::upper_bound(h_tiles, h_tiles + S + 1, t) - h_tiles) - 1;
    const int64_t Ms_i = h_off[i + 1] - h_off[i];
    return h_xoff[i] + std::min((int64_t)(t - h_tiles[i]) * tile, Ms_i) * model->meta[s_first + i].d;
  };
  const int nchunk = (host_src && use_tc) ? std::max(1, std::min(8, tiles / 1024)) : 1;
  if (host_src && nchunk <= 1 && floats_all > 0)
    CK(cudaMemcpyAsync(const_cast<float *>(Xstar_dev), host_src, (size_t)floats_all * 4,
                       cudaMemcpyHostToDevice, ctx->stream));
  if (nchunk > 1 && !ctx->copy_stream) {
    CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (auto &e : ctx->feed_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (tiles == 0) return GPBO_OK;
  if (direct) {
    gpbo::RefineLaunch r{};
    r.meta = p.meta;
    r.Xstar = p.Xstar;
    r.m_off = p.m_off; r.m_base = p.m_base; r.x_off = p.x_off;
    r.best = p.best;
    r.Xs64 = model->Xs64;
    r.ls32 = model->ls32;
    r.alpha64 = model->alpha64;
    r.Linv64 = model->Linv64;
    r.keys = keys_d;
    if (mode != gpbo::kModeArgmax) { r.out_mu = out.mu; r.out_var = out.var; r.out_ei = out.ei; }
    {
      KernTimer t(ctx, kKernFast);
      CK(gpbo::launch_direct(r, S, rows, ctx->stream));
    }
    ctx->launches += 1;
    return GPBO_OK;
  }
  // precise-mean tier (reading R13): float64 mu~ of the candidates of searches whose fit chose
  // it (sf2 |alpha|_1 > kMeanTierL1) -- decided on the device when the fit is still pending
  bool need_mean = false;
  int dmax_raw = 1;
  for (int i = 0; i < S; ++i) {
    const SearchMeta &q = model->meta[s_first + i];
    need_mean = need_mean || model->meta_pending || q.mean_tier;
    dmax_raw = std::max(dmax_raw, q.d);
  }
  static const bool no_tier = getenv("GPBO_NO_MEAN_TIER") != nullptr;  // diagnosis only
  need_mean = need_mean && mode != gpbo::kModePosterior && !no_tier;
  if (need_mean) {
    st = ensure_mean(ctx, (size_t)rows);
    if (st) return st;
    p.mean64 = ctx->mean_d;
  }
  for (int c = 0; c < nchunk && !dense_only; ++c) {
    // (pair: chunk boundaries on whole pair tiles)
    const int ts = pair ? 2 : 1, units = tiles / ts;
    const int ta = ts * (int)((int64_t)units * c / nchunk);
    const int tb = ts * (int)((int64_t)units * (c + 1) / nchunk);
    if (nchunk > 1) {
      // chunk c's rows: from its first tile's row to the next chunk's (the last chunk: to the end)
      const int64_t e0 = c == 0 ? 0 : tile_elem(ta), e1 = tile_elem(tb);
      // no wait before the first copy: the staging buffer's previous users were synchronous
      // calls (finished on return), and the work queued on the stream since (an asynchronous
      // fit) does not touch it -- the copies overlap the fit
      if (e1 > e0)
        CK(cudaMemcpyAsync(const_cast<float *>(Xstar_dev) + e0, host_src + e0,
                           (size_t)(e1 - e0) * 4, cudaMemcpyHostToDevice, ctx->copy_stream));
      CK(cudaEventRecord(ctx->feed_ev[c], ctx->copy_stream));
      CK(cudaStreamWaitEvent(ctx->stream, ctx->feed_ev[c], 0));
    }
    if (need_mean) {
      KernTimer tm(ctx, kKernMean);
      CK(gpbo::launch_mean64(p, model->Xs64, tile, ta, tb - ta, dmax_raw, ctx->mean_d,
                             ctx->etab_d, ctx->num_sms, ctx->stream));
      ctx->launches += 1;
    }
    KernTimer t(ctx, kKernFast);
    if (use_tcs)
      CK(gpbo::launch_score_tcs(p, model->meta.data() + s_first, S, ta, tb - ta, ctx->num_sms,
                                ctx->stream));
    else if (use_tc)
      CK(gpbo::launch_score_tc(p, model->meta.data() + s_first, S, ta, tb - ta, ctx->num_sms,
                               ctx->stream));
    else
      CK(gpbo::launch_score_simt(p, tiles, dmax, nmax, ctx->stream));
    ctx->launches += 1;
  }
  if (mode == gpbo::kModeDebug) return GPBO_OK;
  gpbo::RefineLaunch r{};
  r.meta = p.meta;
  r.Xstar = p.Xstar;
  r.m_off = p.m_off; r.m_base = p.m_base; r.x_off = p.x_off;
  r.best = p.best;
  r.Xs64 = model->Xs64;
  r.ls32 = model->ls32;
  r.alpha64 = model->alpha64;
  r.Linv64 = model->Linv64;
  r.keys = keys_d;
  r.thr = thr_d;
  r.viol = viol_d;
  if (mode == gpbo::kModeArgmax) {
    r.list = ctx->list_d;
    r.list_count = count_d;
  } else {
    r.dense_s = 0;
    r.dense_rows = rows;
    r.dense_var = out.var;
    r.out_mu = out.mu; r.out_var = out.var; r.out_ei = out.ei;
  }
  {
    KernTimer t(ctx, kKernRefine);
    if (dense_only)  // gp_posterior: every row in float64, candidate-tiled
      CK(gpbo::launch_posterior64(r, nmax, dmax_raw, ctx->num_sms, ctx->stream));
    else
      CK(gpbo::launch_refine(r, rows, ctx->num_sms, nmax, ctx->stream));
  }
  ctx->launches += 1;
  return GPBO_OK;
}

// Fast phase + refine + cross-rank max + decode (shared by ei_score_argmax / bo_suggest_batch).
gpbo_status argmax_tail(gpbo_ctx *ctx, const gpbo_model *model, const float *xd,
                        const int64_t *m_off, const int64_t *m_base, const double *best_std,
                        int64_t *idx, float *ei, const float *host_src = nullptr) {
  const int S = model->S;
  gpbo_status st = run_score(ctx, model, 0, S, xd, m_off, m_base, best_std, gpbo::kModeArgmax,
                             Outputs(), host_src);
  if (st) return st;
  unsigned long long *keys_d = ctx->cur_keys_d;
  unsigned long long *viol_d = keys_d + S;
  if (ctx->comm) {  // H10: every rank ends with the same per-search keys (and violation flags)
    NK(ncclAllReduce(keys_d, keys_d, 2 * S, ncclUint64, ncclMax, ctx->comm, ctx->stream));
    ctx->collectives += 1;
  }
  // keys, violations, thresholds and the refine count in one read-back
  CK(cudaMemcpyAsync(ctx->keys_h, keys_d, ctx->cur_key_bytes, cudaMemcpyDeviceToHost,
                     ctx->stream));
  if (model->meta_pending)  // the fit results ride along with the keys
    CK(cudaMemcpyAsync(const_cast<gpbo_model *>(model)->meta.data(), model->meta_d,
                       sizeof(SearchMeta) * S, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  model->meta_pending = false;
  CK(cudaGetLastError());
  harvest_events(ctx);
  ctx->last_refine = (int64_t)((const unsigned int *)(ctx->keys_h + 2 * S))[S];
  // Soundness check of the argmax filter: a refined (or audited) candidate whose float64 EI lies
  // outside its fast-phase bracket means an error bound failed, so the filter may have dropped
  // the true winner.  Such a search is re-scored exactly -- every local row in float64, the
  // oracle's arithmetic -- and, across ranks, combined again (the flags were max-reduced with the
  // keys, so every rank takes the same decision and joins the second all-reduce).
  ctx->last_violations = 0;
  bool any_viol = false;
  for (int s = 0; s < S; ++s) {
    ctx->last_violations += (int64_t)ctx->keys_h[S + s];
    any_viol = any_viol || ctx->keys_h[S + s] != 0ull;
  }
  if (any_viol) {
    gpbo::RefineLaunch r{};
    r.meta = model->meta_d;
    r.Xstar = xd;
    r.m_off = ctx->cur_p_off; r.m_base = ctx->cur_p_off + (S + 1); r.x_off = r.m_base + S;
    r.best = (const double *)(r.x_off + S);
    r.Xs64 = model->Xs64;
    r.ls32 = model->ls32;
    r.alpha64 = model->alpha64;
    r.Linv64 = model->Linv64;
    r.keys = keys_d;
    r.dense_keys = 1;
    for (int s = 0; s < S; ++s) {
      if (ctx->keys_h[S + s] == 0ull) continue;
      const int64_t rows = m_off[s + 1] - m_off[s];
      const SearchMeta &q = model->meta[s];
      CK(cudaMemsetAsync(keys_d + s, 0, 8, ctx->stream));
      if (rows <= 0 || (q.status != GPBO_OK && q.status != GPBO_WDEGENERATE)) continue;
      r.dense_s = s;
      r.dense_rows = rows;
      CK(gpbo::launch_refine(r, rows, ctx->num_sms, model->nmax, ctx->stream));
      ctx->launches += 1;
    }
    if (ctx->comm) {
      NK(ncclAllReduce(keys_d, keys_d, S, ncclUint64, ncclMax, ctx->comm, ctx->stream));
      ctx->collectives += 1;
    }
    CK(cudaMemcpyAsync(ctx->keys_h, keys_d, S * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
  }
  for (int s = 0; s < S; ++s) {
    const unsigned long long k = ctx->keys_h[s];
    const SearchMeta &q = model->meta[s];
    if (k == 0ull) {
      if (idx) idx[s] = -1;
      if (ei) ei[s] = 0.f;
      continue;
    }
    const uint32_t lo = (uint32_t)(k & 0xFFFFFFFFull);
    const uint32_t bits = (uint32_t)(k >> 32);
    float e;
    std::memcpy(&e, &bits, 4);
    if (idx) idx[s] = (int64_t)(0xFFFFFFFFu - lo);
    if (ei) ei[s] = (float)(q.std * (double)e);
  }
  return GPBO_OK;
}

}  // namespace

extern "C" {

const char *gpbo_version(void) {
  return "libgpbo 0.5 (sm_100a; fit fp64 1 CTA or 8/16-CTA cluster/search (multicast G) + O(n^2) "
         "append + ML-II; score: tcgen05 fp16x3 resident (CTA pairs, cta_group::2, for n > 112; "
         "4-deep distance ring for n16 + 16 <= 128) / TMA-streamed, mean on the tensor cores, fp64 "
         "precise-mean tier, fp64 direct for small problems, CUDA-core fallback; fp64 refine with "
         "bracket self-check; fp64 posterior on DMMA; shared-memory candidate generator; host "
         "planner)";
}

gpbo_status gpbo_nccl_unique_id(void *out) {
  if (!out) return GPBO_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return GPBO_ENCCL;
  std::memcpy(out, &id, sizeof(id));
  return GPBO_OK;
}

gpbo_status gpbo_ctx_create(int device, void *cuda_stream, int nranks, int rank,
                            const void *nccl_unique_id, gpbo_ctx **out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) return GPBO_EINVAL;
  if (nranks > 1 && nccl_unique_id == nullptr) return GPBO_EINVAL;
  *out = nullptr;
  gpbo_ctx *ctx = new gpbo_ctx();
  ctx->device = device;
  ctx->stream = (cudaStream_t)cuda_stream;
  ctx->nranks = nranks;
  ctx->rank = rank;
  if (cudaSetDevice(device) != cudaSuccess) { delete ctx; return GPBO_ECUDA; }
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess)
    ctx->num_sms = sms;
  // keep freed model blocks cached in the stream-ordered pool (no device-wide sync per fit)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (const char *e = getenv("GPBO_SCORE_IMPL")) {
    if (!strcmp(e, "simt")) ctx->score_impl = 1;
    if (!strcmp(e, "tc")) ctx->score_impl = 2;
  }
  if (nccl_unique_id != nullptr) {  // (a 1-rank communicator is allowed: same code path)
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    if (ncclCommInitRank(&ctx->comm, nranks, id, rank) != ncclSuccess) {
      delete ctx;
      return GPBO_ENCCL;
    }
  }
  *out = ctx;
  return GPBO_OK;
}

gpbo_status gpbo_ctx_destroy(gpbo_ctx *ctx) {
  if (!ctx) return GPBO_EINVAL;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  for (auto &e : ctx->feed_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->gen_stream) {
    cudaStreamSynchronize(ctx->gen_stream);
    cudaStreamDestroy(ctx->gen_stream);
  }
  if (ctx->gen_ev) cudaEventDestroy(ctx->gen_ev);
  if (ctx->xready_ev) cudaEventDestroy(ctx->xready_ev);
  if (ctx->stage_d) cudaFree(ctx->stage_d);
  if (ctx->aux_d) cudaFree(ctx->aux_d);
  if (ctx->aux_h) cudaFreeHost(ctx->aux_h);
  if (ctx->meta_h) cudaFreeHost(ctx->meta_h);
  if (ctx->meta_ev) cudaEventDestroy(ctx->meta_ev);
  if (ctx->aux_ev) cudaEventDestroy(ctx->aux_ev);
  if (ctx->keys_d) cudaFree(ctx->keys_d);
  if (ctx->keys_h) cudaFreeHost(ctx->keys_h);
  if (ctx->list_d) cudaFree(ctx->list_d);
  if (ctx->mean_d) cudaFree(ctx->mean_d);
  if (ctx->etab_d) cudaFree(ctx->etab_d);
  harvest_events(ctx);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  delete ctx;
  return GPBO_OK;
}

const char *gpbo_last_error(const gpbo_ctx *ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

int64_t gpbo_launch_count(const gpbo_ctx *ctx) { return ctx ? ctx->launches : -1; }

int64_t gpbo_last_refine_count(const gpbo_ctx *ctx) { return ctx ? ctx->last_refine : -1; }

int64_t gpbo_collective_count(const gpbo_ctx *ctx) { return ctx ? ctx->collectives : -1; }

int64_t gpbo_last_ml2_evals(const gpbo_ctx *ctx) { return ctx ? ctx->last_ml2_evals : -1; }

int64_t gpbo_last_bracket_violations(const gpbo_ctx *ctx) {
  return ctx ? ctx->last_violations : -1;
}

gpbo_status gpbo_debug_bound_scale(gpbo_ctx *ctx, float scale) {
  if (!ctx || !std::isfinite(scale)) return GPBO_EINVAL;
  ctx->bound_scale = scale;
  return GPBO_OK;
}

int gpbo_last_score_impl(const gpbo_ctx *ctx) { return ctx ? ctx->last_impl : -1; }
int gpbo_last_tc_pair(const gpbo_ctx *ctx) { return ctx ? ctx->last_pair : -1; }

gpbo_status gpbo_debug_trace(gpbo_ctx *ctx, void *dev_buf) {
  if (!ctx) return GPBO_EINVAL;
  ctx->trace = (unsigned long long *)dev_buf;
  return GPBO_OK;
}

gpbo_status gpbo_set_profiling(gpbo_ctx *ctx, int on) {
  if (!ctx) return GPBO_EINVAL;
  cudaStreamSynchronize(ctx->stream);
  harvest_events(ctx);
  ctx->profiling = on != 0;
  for (int i = 0; i < 5; ++i) { ctx->kern_ms[i] = 0.0; ctx->kern_count[i] = 0; }
  return GPBO_OK;
}

gpbo_status gpbo_kernel_time(gpbo_ctx *ctx, int kind, int64_t *count, double *ms) {
  if (!ctx || kind < 0 || kind > 4) return GPBO_EINVAL;
  cudaStreamSynchronize(ctx->stream);
  harvest_events(ctx);
  if (count) *count = ctx->kern_count[kind];
  if (ms) *ms = ctx->kern_ms[kind];
  return GPBO_OK;
}

gpbo_status gpbo_set_score_impl(gpbo_ctx *ctx, int impl) {
  if (!ctx || impl < 0 || impl > 4) return GPBO_EINVAL;
  ctx->score_impl = impl;
  return GPBO_OK;
}

void gp_model_free(gpbo_model *model) {
  if (!model) return;
  cudaSetDevice(model->device);
  if (model->block) cudaFreeAsync(model->block, model->stream);  // stream-ordered pool
  delete model;
}

namespace {
// Model allocation shared by gp_fit and gp_fit_append: the per-search meta records (shapes,
// offsets, tcgen05 geometry) and one stream-ordered device block holding every array.
struct ModelScratch {
  SearchMeta *meta_in = nullptr;  // device staging of the input meta records
  double *Wscr64 = nullptr, *Kt64 = nullptr, *pm_part = nullptr, *G64 = nullptr;
  int smem_max = 0;
};

gpbo_status alloc_model(gpbo_ctx *ctx, int S, const int32_t *n_in, const int32_t *d_in, int kernel,
                        bool lml_only, gpbo_model **out, ModelScratch *sc) {
  *out = nullptr;
  gpbo_model *m = new gpbo_model();
  m->S = S;
  m->kernel = kernel;
  m->device = ctx->device;
  m->stream = ctx->stream;
  m->meta.resize(S);
  int64_t nx = 0, nls = 0, ny = 0, nmat = 0, nxs = 0, nlt = 0, na = 0, nimg = 0, nscr = 0;
  int64_t nkt = 0, nstg = 0;
  int smem_max = 0;
  // tcgen05 image layout, uniform over the model: streamed (score_tcs.cu) when any search's
  // resident image would not fit in shared memory, or when the ctx forces it (impl 3)
  bool stream_layout = ctx->score_impl == 3;
  for (int s = 0; s < S; ++s)
    if (n_in[s] >= 1 && n_in[s] <= GPBO_MAX_N && d_in[s] >= 1 && d_in[s] <= GPBO_MAX_D &&
        gpbo::tc_needs_stream(n_in[s], d_in[s]))
      stream_layout = true;
  // the CTA-pair scoring layout when every search's resident image fits it (uniform per model)
  bool pair_layout = !stream_layout;
  for (int s = 0; s < S && pair_layout; ++s)
    if (n_in[s] < 1 || n_in[s] > GPBO_MAX_N || d_in[s] < 1 || d_in[s] > GPBO_MAX_D ||
        !gpbo::tc_pair_fits(n_in[s], d_in[s]))
      pair_layout = false;
  for (int s = 0; s < S; ++s) {
    const int n = n_in[s], d = d_in[s];
    if (n < 1 || n > GPBO_MAX_N || d < 1 || d > GPBO_MAX_D) {
      delete m;
      return fail(ctx, GPBO_EINVAL, "n_s must be in [1, 512] and d_s in [1, 64]");
    }
    SearchMeta &q = m->meta[s];
    std::memset(&q, 0, sizeof(q));
    q.n = n;
    q.d = d;
    q.n_pad = (int)round_up(n, 64);
    q.d_pad = (int)round_up(d, 8);
    q.kernel = kernel;
    q.x_off = nx; nx += (int64_t)n * d;
    q.ls_off = nls; nls += d;
    q.y_off = ny; ny += n;
    q.mat_off = nmat; nmat += (int64_t)n * n;
    q.xs_off = nxs; nxs += (int64_t)q.n_pad * q.d_pad;
    q.lt_off = nlt; nlt += (int64_t)q.n_pad * q.n_pad;
    q.a_off = na; na += q.n_pad;
    q.tc_stream = stream_layout ? 1 : 0;
    q.tc_pair = pair_layout ? 1 : 0;
    gpbo::tc_fill_geometry(q);
    q.img_off = nimg;
    if (lml_only) q.tc_ok = 0; else nimg += gpbo::tc_image_bytes(q);
    q.use_smem = n <= gpbo::kFitSmemMaxN;
    if (!q.use_smem) { q.scr_off = nscr; nscr += gpbo::fit_tile_doubles(n); }
    q.kt_off = nkt; nkt += gpbo::fit_tile_doubles(n);
    q.stg_off = nstg; nstg += 16 * gpbo::fit_nr8(n);
    const int smem = gpbo::fit_smem_doubles(n, q.use_smem) * 8;
    q.xs_smem = 0;
    smem_max = std::max(smem_max, smem);
    m->nmax = std::max(m->nmax, n);
    m->dmax = std::max(m->dmax, q.d_pad);
  }
  // one device block: meta | X | ls | Xs | LT | y | L | Linv | alpha | img
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += round_up((int64_t)bytes, 256); return o; };
  const size_t o_meta = take(sizeof(SearchMeta) * S * 2);
  const size_t o_x = take(nx * 4), o_ls = take(nls * 4), o_xs = take(nxs * 4);
  const size_t o_lt = take(nlt * 4), o_y = take(ny * 8), o_L = take(nmat * 8);
  const size_t o_Li = take(nmat * 8), o_a = take(na * 8), o_img = take(nimg);
  const size_t o_x64 = take(nx * 8), o_scr = take(nscr * 8), o_kt = take(nkt * 8);
  const size_t o_pm = take((size_t)S * 16 * 8);
  const size_t o_stg = take((size_t)nstg * 8);
  cudaError_t e = cudaMallocAsync((void **)&m->block, off, ctx->stream);
  if (e != cudaSuccess) { delete m; return fail(ctx, GPBO_ENOMEM, "model allocation failed"); }
  m->meta_d = (SearchMeta *)(m->block + o_meta);
  sc->meta_in = m->meta_d + S;
  m->X32 = (float *)(m->block + o_x);
  m->ls32 = (float *)(m->block + o_ls);
  m->Xs32 = (float *)(m->block + o_xs);
  m->LT32 = (float *)(m->block + o_lt);
  m->y64 = (double *)(m->block + o_y);
  m->L64 = (double *)(m->block + o_L);
  m->Linv64 = (double *)(m->block + o_Li);
  m->alpha64 = (double *)(m->block + o_a);
  m->img = (unsigned char *)(m->block + o_img);
  m->Xs64 = (double *)(m->block + o_x64);
  sc->Wscr64 = (double *)(m->block + o_scr);
  sc->Kt64 = (double *)(m->block + o_kt);
  sc->pm_part = (double *)(m->block + o_pm);
  sc->G64 = (double *)(m->block + o_stg);
  sc->smem_max = smem_max;
  m->img_bytes = nimg;
  m->nx_total = nx; m->nls_total = nls; m->ny_total = ny;
  *out = m;
  return GPBO_OK;
}

// CTAs per search of the cluster fit, or 0 for the one-CTA kernel (GPBO_FIT=single)
int fit_cluster_size(const gpbo_ctx *ctx, int S, int nmax) {
  static const bool single = [] {
    const char *e = getenv("GPBO_FIT");
    return e && !strcmp(e, "single");
  }();
  static const bool force_cluster = [] {  // A/B: the cluster fit for every n
    const char *e = getenv("GPBO_FIT");
    return e && !strcmp(e, "cluster");
  }();
  // measured (profiles/r02): for n <= 216 the one-CTA kernel keeps its working matrix in shared
  // memory and the cluster's DSMEM hops (~2.5 k cycles per panel) cost as much as the split
  // trailing update saves (n = 200: 0.139 vs 0.140 ms; 64 x n = 100: 0.056 vs 0.084 ms); for
  // n > 216 the one-CTA kernel streams W through L2 and the cluster wins (n = 500: 1.27 -> 0.68 ms)
  if (single || (nmax <= gpbo::kFitSmemMaxN && !force_cluster)) return 0;
  const int per = ctx->num_sms / std::max(S, 1);
  int Cc = per >= 16 ? 16 : per >= 8 ? 8 : per >= 4 ? 4 : per >= 2 ? 2 : 1;
  static const int cc_cap = [] {  // A/B: cap the cluster size (GPBO_FIT_CC=1|2|4|8|16)
    const char *e = getenv("GPBO_FIT_CC");
    return e ? atoi(e) : 16;
  }();
  if (cc_cap >= 1 && cc_cap < Cc) Cc = cc_cap;
  // 16-CTA (non-portable) clusters: only where the device can hold one at this size
  if (Cc == 16 && !gpbo::fit_cluster16_ok(gpbo::fit_cluster_smem(nmax, 16))) Cc = 8;
  while (Cc < 8 && gpbo::fit_cluster_smem(nmax, Cc) > gpbo::kFitSmemBudget) Cc *= 2;
  return gpbo::fit_cluster_smem(nmax, Cc) <= gpbo::kFitSmemBudget ? Cc : 0;
}

// lml_only (ML-II objective evaluations): no tcgen05 operand image is reserved; the model is
// read for its statistics and freed, never scored.
gpbo_status fit_impl(gpbo_ctx *ctx, const gpbo_fit_args *a, gpbo_model **out, bool wait,
                     int32_t *status, int32_t *jitter_k, bool lml_only = false) {
  if (!ctx) return GPBO_EINVAL;
  if (!a || !out) return fail(ctx, GPBO_EINVAL, "null args/out");
  *out = nullptr;
  if (a->S < 1 || !a->n || !a->d || !a->X || !a->y || !a->lengthscale || !a->signal_var ||
      !a->noise_var)
    return fail(ctx, GPBO_EINVAL, "S < 1 or null input array");
  if (a->kernel != GPBO_RBF && a->kernel != GPBO_MATERN52)
    return fail(ctx, GPBO_EINVAL, "unknown kernel");
  if (a->mem != GPBO_HOST && a->mem != GPBO_DEVICE) return fail(ctx, GPBO_EINVAL, "bad mem");
  CK(cudaSetDevice(ctx->device));
  const int S = a->S;
  gpbo_model *m = nullptr;
  ModelScratch sc;
  {
    gpbo_status ast = alloc_model(ctx, S, a->n, a->d, a->kernel, lml_only, &m, &sc);
    if (ast) return ast;
  }
  SearchMeta *meta_in = sc.meta_in;
  double *Wscr64 = sc.Wscr64, *Kt64 = sc.Kt64;
  const int smem_max = sc.smem_max;
  const int64_t nx = m->nx_total, nls = m->nls_total, ny = m->ny_total;
  // hyper-parameters: host arrays go into the meta records; device arrays are read by the kernel
  if (a->mem == GPBO_HOST)
    for (int s = 0; s < S; ++s) { m->meta[s].sf2 = a->signal_var[s]; m->meta[s].sn2 = a->noise_var[s]; }
  const cudaMemcpyKind kind = a->mem == GPBO_HOST ? cudaMemcpyHostToDevice
                                                  : cudaMemcpyDeviceToDevice;
  auto cleanup_fail = [&](gpbo_status st, const std::string &msg) {
    cudaStreamSynchronize(ctx->stream);
    gp_model_free(m);
    return fail(ctx, st, msg);
  };
#define CKM(x)                                                                          \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      return cleanup_fail(GPBO_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
  gpbo::FitIO io{};
  io.X32 = m->X32; io.ls32 = m->ls32; io.y64 = m->y64;
  io.L64 = m->L64; io.Linv64 = m->Linv64; io.Xs64 = m->Xs64; io.alpha64 = m->alpha64;
  io.Wscr64 = Wscr64;
  io.Kt64 = Kt64;
  io.pm_part = sc.pm_part;
  io.G64 = sc.G64;
  if (a->mem == GPBO_HOST) {  // stage into the model's arrays
    CKM(cudaMemcpyAsync(m->X32, a->X, nx * 4, kind, ctx->stream));
    CKM(cudaMemcpyAsync(m->ls32, a->lengthscale, nls * 4, kind, ctx->stream));
    CKM(cudaMemcpyAsync(m->y64, a->y, ny * 8, kind, ctx->stream));
    io.X_src = m->X32; io.ls_src = m->ls32; io.y_src = m->y64;
  } else {  // the kernel reads the caller's arrays and copies them
    io.X_src = a->X; io.ls_src = a->lengthscale; io.y_src = a->y;
    io.sf2_src = a->signal_var; io.sn2_src = a->noise_var;
  }
  gpbo_status pst = ensure_meta_h(ctx, sizeof(SearchMeta) * S);
  if (pst) { gp_model_free(m); return pst; }
  if (ctx->meta_ev) CKM(cudaEventSynchronize(ctx->meta_ev));  // previous upload read meta_h
  std::memcpy(ctx->meta_h, m->meta.data(), sizeof(SearchMeta) * S);
  CKM(cudaMemcpyAsync(meta_in, ctx->meta_h, sizeof(SearchMeta) * S, cudaMemcpyHostToDevice,
                      ctx->stream));
  if (!ctx->meta_ev) CKM(cudaEventCreateWithFlags(&ctx->meta_ev, cudaEventDisableTiming));
  CKM(cudaEventRecord(ctx->meta_ev, ctx->stream));
  {
    KernTimer t(ctx, kKernFit);
    CKM(gpbo::launch_gram(meta_in, S, m->nmax, m->dmax, io, ctx->stream));
    // the model's X32 is complete once the pre-pass has run (bo_suggest_batch's dedup reads it)
    if (!ctx->xready_ev) CKM(cudaEventCreateWithFlags(&ctx->xready_ev, cudaEventDisableTiming));
    CKM(cudaEventRecord(ctx->xready_ev, ctx->stream));
    // the factorisation: a cluster of Cc CTAs per search (fit_cluster.cu) -- as many CTAs per
    // search as the SMs allow (~148 / S), and enough that the distributed working matrix fits in
    // their shared memory; GPBO_FIT=single selects the one-CTA kernel (fit.cu) for A/B runs
    const int Cc = fit_cluster_size(ctx, S, m->nmax);
    // (packing the scoring image in the one-CTA fit's tail, io.img, measured 52 us slower than
    // the 64-CTA pack kernel's 15 us at n = 200: one SM converting 129 KB; kept off)
    io.img = nullptr;
    if (Cc > 0)
      CKM(gpbo::launch_fit_cluster(meta_in, S, Cc, gpbo::fit_cluster_smem(m->nmax, Cc), io,
                                   m->meta_d, ctx->stream));
    else
      CKM(gpbo::launch_fit(meta_in, S, smem_max, io, m->meta_d, ctx->stream,
                           m->nmax <= gpbo::kFitSmemMaxN));
  }
  ctx->launches += 2;  // gram_kernel + fit_kernel
  // the tcgen05 operand images are packed by the first tcgen05 scoring call (run_score): small
  // problems scored by the float64 direct kernel never need them
  if (!wait) {  // gp_fit_async: results stay on the device until gp_model_sync / scoring
    m->meta_pending = true;
    *out = m;
    return GPBO_OK;
  }
  CKM(cudaMemcpyAsync(ctx->meta_h, m->meta_d, sizeof(SearchMeta) * S, cudaMemcpyDeviceToHost,
                      ctx->stream));
  CKM(cudaStreamSynchronize(ctx->stream));
  std::memcpy(m->meta.data(), ctx->meta_h, sizeof(SearchMeta) * S);
  harvest_events(ctx);
#undef CKM
  gpbo_status worst = GPBO_OK;
  bool einval = false;
  for (int s = 0; s < S; ++s) {
    const SearchMeta &q = m->meta[s];
    if (status) status[s] = q.status;
    if (jitter_k) jitter_k[s] = q.jitter_k;
    if (q.status == GPBO_EINVAL) einval = true;
    if (q.status == GPBO_ENOTPD) worst = GPBO_ENOTPD;
    else if (q.status == GPBO_WDEGENERATE && worst == GPBO_OK) worst = GPBO_WDEGENERATE;
  }
  if (einval) {
    gp_model_free(m);
    return fail(ctx, GPBO_EINVAL, "non-finite or out-of-domain fit input");
  }
  *out = m;
  if (worst == GPBO_ENOTPD) ctx->err = "Cholesky failed at the largest jitter for some search";
  return worst;
}
}  // namespace

gpbo_status gp_fit(gpbo_ctx *ctx, const gpbo_fit_args *a, gpbo_model **out, int32_t *status,
                   int32_t *jitter_k) {
  return fit_impl(ctx, a, out, true, status, jitter_k);
}

gpbo_status gpbo_nm_selftest(int dim, const double *x0, const double *lo, const double *hi,
                             double step, int iters, double (*f)(const double *x, void *user),
                             void *user, double *best_x, double *best_f, double *start_f,
                             int64_t *nevals) {
  if (dim < 1 || !x0 || !lo || !hi || !f || !best_x || !(step > 0) || iters < 0)
    return GPBO_EINVAL;
  gpbo::NelderMead nm(dim, x0, lo, hi, step, iters);
  int64_t ne = 0;
  std::vector<double> fv;
  while (!nm.done()) {
    const std::vector<double> &req = nm.request();
    const int np = (int)(req.size() / dim);
    fv.resize(np);
    for (int p = 0; p < np; ++p) fv[p] = f(&req[(size_t)p * dim], user);
    ne += np;
    nm.deliver(fv.data());
  }
  for (int i = 0; i < dim; ++i) best_x[i] = nm.best_x()[i];
  if (best_f) *best_f = nm.best_f();
  if (start_f) *start_f = nm.start_f();
  if (nevals) *nevals = ne;
  return GPBO_OK;
}

gpbo_status gp_fit_append(gpbo_ctx *ctx, const gpbo_model *prev, const float *x_new,
                          const double *y_new, gpbo_mem mem, gpbo_model **out, int32_t *status,
                          int32_t *jitter_k) {
  if (!ctx) return GPBO_EINVAL;
  if (!prev || !x_new || !y_new || !out) return fail(ctx, GPBO_EINVAL, "null argument");
  *out = nullptr;
  if (mem != GPBO_HOST && mem != GPBO_DEVICE) return fail(ctx, GPBO_EINVAL, "bad mem");
  CK(cudaSetDevice(ctx->device));
  if (refresh_meta(prev)) return fail(ctx, GPBO_ECUDA, "meta download failed");
  const int S = prev->S;
  std::vector<int32_t> n1(S), d(S);
  int64_t dsum = 0;
  for (int s = 0; s < S; ++s) {
    const SearchMeta &q = prev->meta[s];
    if (q.status != GPBO_OK && q.status != GPBO_WDEGENERATE)
      return fail(ctx, GPBO_EINVAL, "gp_fit_append: a search of the previous model has no fit");
    if (q.n + 1 > GPBO_MAX_N) return fail(ctx, GPBO_EINVAL, "gp_fit_append: n would exceed 512");
    n1[s] = q.n + 1;
    d[s] = q.d;
    dsum += q.d;
  }
  gpbo_model *m = nullptr;
  ModelScratch sc;
  gpbo_status st = alloc_model(ctx, S, n1.data(), d.data(), prev->kernel, false, &m, &sc);
  if (st) return st;
  for (int s = 0; s < S; ++s) { m->meta[s].sf2 = prev->meta[s].sf2; m->meta[s].sn2 = prev->meta[s].sn2; }
  auto cleanup_fail = [&](gpbo_status e, const std::string &msg) {
    cudaStreamSynchronize(ctx->stream);
    gp_model_free(m);
    return fail(ctx, e, msg);
  };
#define CKA(x)                                                                          \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      return cleanup_fail(GPBO_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
  // new observations: host values staged through the scratch the fit would use (Kt64, unused
  // by an appended model), device values read in place
  const float *xd = x_new;
  const double *yd = y_new;
  if (mem == GPBO_HOST) {
    gpbo_status e = ensure_stage(ctx, (size_t)dsum * 4 + (size_t)S * 8 + 64);
    if (e) { gp_model_free(m); return e; }
    double *ys = (double *)ctx->stage_d;
    float *xs = (float *)(ys + S);
    CKA(cudaMemcpyAsync(ys, y_new, (size_t)S * 8, cudaMemcpyHostToDevice, ctx->stream));
    CKA(cudaMemcpyAsync(xs, x_new, (size_t)dsum * 4, cudaMemcpyHostToDevice, ctx->stream));
    xd = xs;
    yd = ys;
  }
  gpbo_status pst = ensure_meta_h(ctx, sizeof(SearchMeta) * S);
  if (pst) { gp_model_free(m); return pst; }
  if (ctx->meta_ev) CKA(cudaEventSynchronize(ctx->meta_ev));
  std::memcpy(ctx->meta_h, m->meta.data(), sizeof(SearchMeta) * S);
  CKA(cudaMemcpyAsync(sc.meta_in, ctx->meta_h, sizeof(SearchMeta) * S, cudaMemcpyHostToDevice,
                      ctx->stream));
  if (!ctx->meta_ev) CKA(cudaEventCreateWithFlags(&ctx->meta_ev, cudaEventDisableTiming));
  CKA(cudaEventRecord(ctx->meta_ev, ctx->stream));
  gpbo::AppendIO io{};
  io.prev_meta = prev->meta_d;
  io.prev_X32 = prev->X32; io.prev_ls32 = prev->ls32; io.prev_y64 = prev->y64;
  io.prev_L64 = prev->L64; io.prev_Linv64 = prev->Linv64; io.prev_Xs64 = prev->Xs64;
  io.x_new = xd; io.y_new = yd;
  io.X32 = m->X32; io.ls32 = m->ls32; io.y64 = m->y64; io.L64 = m->L64;
  io.Linv64 = m->Linv64; io.Xs64 = m->Xs64; io.alpha64 = m->alpha64;
  {
    KernTimer t(ctx, kKernFit);
    CKA(gpbo::launch_append(sc.meta_in, S, io, m->meta_d, ctx->stream));
  }
  ctx->launches += 1;
  CKA(cudaMemcpyAsync(ctx->meta_h, m->meta_d, sizeof(SearchMeta) * S, cudaMemcpyDeviceToHost,
                      ctx->stream));
  CKA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(m->meta.data(), ctx->meta_h, sizeof(SearchMeta) * S);
  harvest_events(ctx);
#undef CKA
  bool einval = false, refit = false;
  for (int s = 0; s < S; ++s) {
    einval = einval || m->meta[s].status == GPBO_EINVAL;
    refit = refit || (m->meta[s].status == GPBO_ENOTPD && m->meta[s].jitter_k == -2);
  }
  if (einval) {
    gp_model_free(m);
    return fail(ctx, GPBO_EINVAL, "non-finite new observation");
  }
  ctx->last_append_refit = refit ? 1 : 0;
  if (refit) {
    // the bordered matrix is not positive definite at the old jitter: refit every search from
    // the appended data (already on the device) with the full jitter ladder
    std::vector<float> sf2(S), sn2(S);
    for (int s = 0; s < S; ++s) { sf2[s] = prev->meta[s].sf2; sn2[s] = prev->meta[s].sn2; }
    // device hyper-parameter arrays for the device-input fit: staged after the new data
    gpbo_status e = ensure_stage(ctx, (size_t)S * 8 + 64);
    if (e) { gp_model_free(m); return e; }
    float *hp = (float *)ctx->stage_d;
    if (cudaMemcpyAsync(hp, sf2.data(), (size_t)S * 4, cudaMemcpyHostToDevice, ctx->stream) ||
        cudaMemcpyAsync(hp + S, sn2.data(), (size_t)S * 4, cudaMemcpyHostToDevice, ctx->stream)) {
      gp_model_free(m);
      return fail(ctx, GPBO_ECUDA, "staging failed");
    }
    gpbo_fit_args fa{};
    fa.S = S; fa.n = n1.data(); fa.d = d.data(); fa.X = m->X32; fa.y = m->y64;
    fa.lengthscale = m->ls32; fa.signal_var = hp; fa.noise_var = hp + S;
    fa.kernel = (gpbo_kernel)prev->kernel; fa.mem = GPBO_DEVICE;
    gpbo_model *r = nullptr;
    st = fit_impl(ctx, &fa, &r, true, status, jitter_k);  // synchronous: m's arrays are read
    gp_model_free(m);
    if (r) *out = r;
    return st;
  }
  gpbo_status worst = GPBO_OK;
  for (int s = 0; s < S; ++s) {
    if (status) status[s] = m->meta[s].status;
    if (jitter_k) jitter_k[s] = m->meta[s].jitter_k;
    if (m->meta[s].status == GPBO_WDEGENERATE) worst = GPBO_WDEGENERATE;
  }
  *out = m;
  return worst;
}

int64_t gpbo_last_append_refit(const gpbo_ctx *ctx) { return ctx ? ctx->last_append_refit : -1; }

gpbo_status gp_model_lml(const gpbo_model *model, double *lml) {
  if (!model || !lml) return GPBO_EINVAL;
  if (refresh_meta(model)) return GPBO_ECUDA;
  for (int s = 0; s < model->S; ++s) lml[s] = model->meta[s].lml;
  return GPBO_OK;
}

gpbo_status gp_fit_ml2(gpbo_ctx *ctx, const gpbo_fit_args *a, const gpbo_ml2_opts *opt,
                       float *ls_out, float *sf2_out, float *sn2_out, double *lml_out,
                       double *lml_starts) {
  if (!ctx) return GPBO_EINVAL;
  if (!a || !opt || !ls_out || !sf2_out || !sn2_out)
    return fail(ctx, GPBO_EINVAL, "null args/opts/outputs");
  if (a->mem != GPBO_HOST) return fail(ctx, GPBO_EINVAL, "gp_fit_ml2 takes host inputs");
  if (a->S < 1 || !a->n || !a->d || !a->X || !a->y || !a->lengthscale || !a->signal_var ||
      !a->noise_var)
    return fail(ctx, GPBO_EINVAL, "S < 1 or null input array");
  if (opt->starts < 1 || opt->iters < 0 || !(opt->ls_lo > 0) || !(opt->ls_hi >= opt->ls_lo) ||
      !(opt->sf2_lo > 0) || !(opt->sf2_hi >= opt->sf2_lo) || !(opt->sn2_lo > 0) ||
      !(opt->sn2_hi >= opt->sn2_lo) || !(opt->step > 0))
    return fail(ctx, GPBO_EINVAL, "bad ML-II options");
  const int S = a->S, K = opt->starts;
  std::vector<int64_t> xo(S + 1, 0), yo(S + 1, 0), lo_(S + 1, 0);
  for (int s = 0; s < S; ++s) {
    if (a->n[s] < 1 || a->n[s] > GPBO_MAX_N || a->d[s] < 1 || a->d[s] > GPBO_MAX_D)
      return fail(ctx, GPBO_EINVAL, "n_s must be in [1, 512] and d_s in [1, 64]");
    xo[s + 1] = xo[s] + (int64_t)a->n[s] * a->d[s];
    yo[s + 1] = yo[s] + a->n[s];
    lo_[s + 1] = lo_[s] + a->d[s];
  }
  // theta of search s in log space: (log l_1 .. log l_d, log sf2, log sn2), dim d + 2
  std::vector<gpbo::NelderMead> lanes;
  std::vector<int> lane_s;
  lanes.reserve((size_t)S * K);
  for (int s = 0; s < S; ++s) {
    const int d = a->d[s], dim = d + 2;
    std::vector<double> lo(dim), hi(dim), x0(dim);
    for (int i = 0; i < d; ++i) { lo[i] = std::log(opt->ls_lo); hi[i] = std::log(opt->ls_hi); }
    lo[d] = std::log(opt->sf2_lo); hi[d] = std::log(opt->sf2_hi);
    lo[d + 1] = std::log(opt->sn2_lo); hi[d + 1] = std::log(opt->sn2_hi);
    for (int k = 0; k < K; ++k) {
      if (k == 0) {  // start 0: the caller's theta
        for (int i = 0; i < d; ++i) x0[i] = std::log((double)a->lengthscale[lo_[s] + i]);
        x0[d] = std::log((double)a->signal_var[s]);
        x0[d + 1] = std::log((double)a->noise_var[s]);
        for (int i = 0; i < dim; ++i)
          if (!std::isfinite(x0[i])) return fail(ctx, GPBO_EINVAL, "start theta must be > 0");
      } else {  // seeded uniform starts in the log box
        for (int i = 0; i < dim; ++i)
          x0[i] = lo[i] + gpbo::ml2_uniform(opt->seed, s, k, i, dim, K) * (hi[i] - lo[i]);
      }
      lanes.emplace_back(dim, x0.data(), lo.data(), hi.data(), opt->step, opt->iters);
      lane_s.push_back(s);
    }
  }
  // rounds: every unfinished simplex contributes its requested points to one batched fit
  std::vector<int32_t> bn, bd;
  std::vector<float> bX, bls, bsf2, bsn2;
  std::vector<double> by, fvals;
  std::vector<std::pair<int, int>> owner;  // (lane, point count) per lane in the batch
  int64_t evals = 0;
  for (;;) {
    bn.clear(); bd.clear(); bX.clear(); bls.clear(); bsf2.clear(); bsn2.clear(); by.clear();
    owner.clear();
    for (size_t l = 0; l < lanes.size(); ++l) {
      if (lanes[l].done()) continue;
      const int s = lane_s[l], d = a->d[s], dim = d + 2;
      const std::vector<double> &req = lanes[l].request();
      const int np = (int)(req.size() / dim);
      for (int p = 0; p < np; ++p) {
        const double *x = &req[(size_t)p * dim];
        bn.push_back(a->n[s]);
        bd.push_back(d);
        bX.insert(bX.end(), a->X + xo[s], a->X + xo[s + 1]);
        by.insert(by.end(), a->y + yo[s], a->y + yo[s + 1]);
        for (int i = 0; i < d; ++i) bls.push_back((float)std::exp(x[i]));
        bsf2.push_back((float)std::exp(x[d]));
        bsn2.push_back((float)std::exp(x[d + 1]));
      }
      owner.push_back({(int)l, np});
    }
    if (owner.empty()) break;
    gpbo_fit_args fa{};
    fa.S = (int32_t)bn.size();
    fa.n = bn.data(); fa.d = bd.data(); fa.X = bX.data(); fa.y = by.data();
    fa.lengthscale = bls.data(); fa.signal_var = bsf2.data(); fa.noise_var = bsn2.data();
    fa.kernel = a->kernel; fa.mem = GPBO_HOST;
    gpbo_model *m = nullptr;
    gpbo_status st = fit_impl(ctx, &fa, &m, true, nullptr, nullptr, true);
    if (st != GPBO_OK && st != GPBO_ENOTPD && st != GPBO_WDEGENERATE) {
      if (m) gp_model_free(m);
      return st;
    }
    evals += fa.S;
    int q = 0;
    for (auto &o : owner) {
      fvals.assign(o.second, 0.0);
      for (int p = 0; p < o.second; ++p, ++q) {
        const SearchMeta &r = m->meta[q];
        const bool ok = (r.status == GPBO_OK || r.status == GPBO_WDEGENERATE) && std::isfinite(r.lml);
        fvals[p] = ok ? -r.lml : INFINITY;  // minimise -LML
      }
      lanes[o.first].deliver(fvals.data());
    }
    gp_model_free(m);
  }
  ctx->last_ml2_evals = evals;
  // per search: the best vertex over its starts (ties -> the lowest start)
  for (int s = 0; s < S; ++s) {
    const int d = a->d[s];
    int bl = s * K;
    for (int k = 0; k < K; ++k) {
      const int l = s * K + k;
      if (lanes[l].best_f() < lanes[bl].best_f()) bl = l;
      if (lml_starts) lml_starts[(size_t)s * K + k] = -lanes[l].start_f();
    }
    const double *x = lanes[bl].best_x();
    for (int i = 0; i < d; ++i) ls_out[lo_[s] + i] = (float)std::exp(x[i]);
    sf2_out[s] = (float)std::exp(x[d]);
    sn2_out[s] = (float)std::exp(x[d + 1]);
    if (lml_out) lml_out[s] = -lanes[bl].best_f();
  }
  return GPBO_OK;
}

gpbo_status gp_fit_async(gpbo_ctx *ctx, const gpbo_fit_args *a, gpbo_model **out) {
  return fit_impl(ctx, a, out, false, nullptr, nullptr);
}

gpbo_status gp_model_sync(gpbo_ctx *ctx, const gpbo_model *model, int32_t *status,
                          int32_t *jitter_k) {
  if (!ctx) return GPBO_EINVAL;
  if (!model) return fail(ctx, GPBO_EINVAL, "null model");
  if (refresh_meta(model)) return fail(ctx, GPBO_ECUDA, "meta download failed");
  gpbo_status worst = GPBO_OK;
  for (int s = 0; s < model->S; ++s) {
    const SearchMeta &q = model->meta[s];
    if (status) status[s] = q.status;
    if (jitter_k) jitter_k[s] = q.jitter_k;
    if (q.status == GPBO_EINVAL) worst = GPBO_EINVAL;
    else if (q.status == GPBO_ENOTPD && worst != GPBO_EINVAL) worst = GPBO_ENOTPD;
    else if (q.status == GPBO_WDEGENERATE && worst == GPBO_OK) worst = GPBO_WDEGENERATE;
  }
  return worst;
}

gpbo_status gp_model_stats(const gpbo_model *model, int32_t s, double *mean, double *std,
                           double *best, double *alpha_l1) {
  if (!model || s < 0 || s >= model->S) return GPBO_EINVAL;
  if (refresh_meta(model)) return GPBO_ECUDA;
  const SearchMeta &q = model->meta[s];
  if (mean) *mean = q.mean;
  if (std) *std = q.std;
  if (best) *best = q.best;
  if (alpha_l1) *alpha_l1 = q.alpha_l1;
  return GPBO_OK;
}

gpbo_status gp_model_export(gpbo_ctx *ctx, const gpbo_model *model, int32_t s, double *L,
                            double *Linv, double *alpha) {
  if (!ctx) return GPBO_EINVAL;
  if (model && refresh_meta(model)) return fail(ctx, GPBO_ECUDA, "meta download failed");
  if (!model || s < 0 || s >= model->S) return fail(ctx, GPBO_EINVAL, "bad model/search");
  CK(cudaSetDevice(ctx->device));
  const SearchMeta &q = model->meta[s];
  const int n = q.n;
  std::vector<double> buf((size_t)n * n);
  double *outs[2] = {L, Linv};
  double *srcs[2] = {model->L64, model->Linv64};
  for (int w = 0; w < 2; ++w) {
    if (!outs[w]) continue;
    CK(cudaMemcpyAsync(buf.data(), srcs[w] + q.mat_off, buf.size() * 8, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int j = 0; j < n; ++j)  // device lower part (L col-major, L^-1 row-major) -> row-major
      for (int i = 0; i < n; ++i)
        outs[w][(size_t)i * n + j] = i < j ? 0.0 : w == 0 ? buf[(size_t)j * n + i] : buf[(size_t)i * n + j];
  }
  if (alpha) {
    CK(cudaMemcpyAsync(alpha, model->alpha64 + q.a_off, n * 8, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return GPBO_OK;
}

gpbo_status gp_posterior(gpbo_ctx *ctx, const gpbo_model *model, int32_t s, const float *Xstar,
                         int64_t M, gpbo_mem mem, float *mu, float *var, float *ei) {
  if (!ctx) return GPBO_EINVAL;
  if (!model || s < 0 || s >= model->S || M < 0 || (M > 0 && !Xstar))
    return fail(ctx, GPBO_EINVAL, "bad model/search/candidates");
  if (mem != GPBO_HOST && mem != GPBO_DEVICE) return fail(ctx, GPBO_EINVAL, "bad mem");
  CK(cudaSetDevice(ctx->device));
  if (refresh_meta(model)) return fail(ctx, GPBO_ECUDA, "meta download failed");
  const SearchMeta &q = model->meta[s];
  if (q.status != GPBO_OK && q.status != GPBO_WDEGENERATE)
    return fail(ctx, GPBO_ENOTPD, "search has no valid fit");
  if (M == 0) return GPBO_OK;
  // device staging: [X* if host] | mu | var | ei  (var is always needed by the refine pass)
  const size_t xb = mem == GPBO_HOST ? round_up((int64_t)M * q.d * 4, 256) : 0;
  const size_t ob = round_up(M * 4, 256);
  gpbo_status st = ensure_stage(ctx, xb + 3 * ob);
  if (st) return st;
  char *b = (char *)ctx->stage_d;
  const float *xd = Xstar;
  if (mem == GPBO_HOST) {
    CK(cudaMemcpyAsync(b, Xstar, (size_t)M * q.d * 4, cudaMemcpyHostToDevice, ctx->stream));
    xd = (const float *)b;
  }
  Outputs o;
  o.mu = (mem == GPBO_DEVICE && mu) ? mu : (float *)(b + xb);
  o.var = (mem == GPBO_DEVICE && var) ? var : (float *)(b + xb + ob);
  o.ei = (mem == GPBO_DEVICE && ei) ? ei : (float *)(b + xb + 2 * ob);
  const int64_t off[2] = {0, M};
  const double best = NAN;  // the fitted incumbent (resolved on the device)
  st = run_score(ctx, model, s, 1, xd, off, nullptr, &best, gpbo::kModePosterior, o);
  if (st) return st;
  if (mem == GPBO_HOST) {
    if (mu) CK(cudaMemcpyAsync(mu, o.mu, M * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (var) CK(cudaMemcpyAsync(var, o.var, M * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (ei) CK(cudaMemcpyAsync(ei, o.ei, M * 4, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaGetLastError());
  return GPBO_OK;
}

gpbo_status gpbo_debug_fast_phase(gpbo_ctx *ctx, const gpbo_model *model, int32_t s,
                                  const float *Xstar_dev, int64_t M, float *mu, float *dmu,
                                  float *var, float *dvar, float *ei_lo, float *ei_hi) {
  if (!ctx) return GPBO_EINVAL;
  if (!model || s < 0 || s >= model->S || M <= 0 || !Xstar_dev || !mu || !dmu || !var ||
      !dvar || !ei_lo || !ei_hi)
    return fail(ctx, GPBO_EINVAL, "bad debug arguments (device arrays required)");
  CK(cudaSetDevice(ctx->device));
  Outputs o;
  float *d[6] = {mu, dmu, var, dvar, ei_lo, ei_hi};
  for (int i = 0; i < 6; ++i) o.dbg[i] = d[i];
  const int64_t off[2] = {0, M};
  if (refresh_meta(model)) return fail(ctx, GPBO_ECUDA, "meta download failed");
  const double best = NAN;  // the fitted incumbent (resolved on the device)
  gpbo_status st = run_score(ctx, model, s, 1, Xstar_dev, off, nullptr, &best,
                             gpbo::kModeDebug, o);
  if (st) return st;
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaGetLastError());
  return GPBO_OK;
}

gpbo_status ei_score_argmax(gpbo_ctx *ctx, const gpbo_model *model, const float *Xstar,
                            const int64_t *m_off, const int64_t *m_global_base,
                            const double *best, gpbo_mem mem, int64_t *idx, float *ei) {
  if (!ctx) return GPBO_EINVAL;
  if (!model || !m_off) return fail(ctx, GPBO_EINVAL, "null model/m_off");
  if (mem != GPBO_HOST && mem != GPBO_DEVICE) return fail(ctx, GPBO_EINVAL, "bad mem");
  CK(cudaSetDevice(ctx->device));
  const int S = model->S;
  std::vector<double> best_std(S);
  int64_t rows = 0, floats = 0;
  for (int s = 0; s < S; ++s) {
    const SearchMeta &q = model->meta[s];
    best_std[s] = best ? best[s] : NAN;  // raw units (standardised on the device) / fitted best
    const int64_t Ms = m_off[s + 1] - m_off[s];
    if (Ms < 0) return fail(ctx, GPBO_EINVAL, "m_off must be non-decreasing");
    rows += Ms;
    floats += Ms * q.d;
  }
  if (rows > 0 && !Xstar) return fail(ctx, GPBO_EINVAL, "null Xstar");
  // rows of search s start at element sum_{t<s} (m_off[t+1] - m_off[t]) d_t of Xstar
  // host candidates: copied into the staging buffer by run_score (chunked, overlapped with the
  // scoring of the previous chunk)
  const float *xd = Xstar, *host_src = nullptr;
  if (mem == GPBO_HOST && floats > 0) {
    gpbo_status st = ensure_stage(ctx, (size_t)floats * 4);
    if (st) return st;
    host_src = Xstar;
    xd = (const float *)ctx->stage_d;
  }
  return argmax_tail(ctx, model, xd, m_off, m_global_base, best_std.data(), idx, ei, host_src);
}

gpbo_status gpbo_space_sample(gpbo_ctx *ctx, const gpbo_space *space, uint64_t seed,
                              int32_t search, int32_t iteration, int64_t first_idx,
                              int64_t count, gpbo_mem mem, float *enc) {
  if (!ctx) return GPBO_EINVAL;
  if (!space || !enc || count < 0 || first_idx < 0 || first_idx + count > 0xFFFFFFFFll)
    return fail(ctx, GPBO_EINVAL, "bad space/sample arguments");
  CK(cudaSetDevice(ctx->device));
  const int d = gpbo_space_dim(space);
  float *out = enc;
  if (mem == GPBO_HOST) {
    gpbo_status st = ensure_stage(ctx, (size_t)count * d * 4 + 16);
    if (st) return st;
    out = (float *)ctx->stage_d;
  }
  CK(gpbo::launch_gen(gpbo::space_dev(space), seed, (uint32_t)search, (uint32_t)iteration,
                      first_idx, count, out, nullptr, 0, ctx->stream));
  ctx->launches += 1;
  if (mem == GPBO_HOST)
    CK(cudaMemcpyAsync(enc, out, (size_t)count * d * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return GPBO_OK;
}

gpbo_status bo_suggest_batch(gpbo_ctx *ctx, const gpbo_model *model,
                             const gpbo_space *const *spaces, const int64_t *M, uint64_t seed,
                             int32_t iteration, int32_t dedup, int64_t *idx, double *x_raw,
                             float *ei) {
  if (!ctx) return GPBO_EINVAL;
  if (!model || !spaces || !M) return fail(ctx, GPBO_EINVAL, "null model/spaces/M");
  CK(cudaSetDevice(ctx->device));
  const int S = model->S;
  std::vector<int64_t> off(S + 1, 0), base(S, 0), xoff(S + 1, 0);
  std::vector<double> best_std(S);
  for (int s = 0; s < S; ++s) {
    if (!spaces[s] || gpbo_space_dim(spaces[s]) != model->meta[s].d)
      return fail(ctx, GPBO_EINVAL, "space dimension does not match the model");
    if (M[s] < 0 || M[s] >= 0xFFFFFFFFll) return fail(ctx, GPBO_EINVAL, "bad pool size");
    const int64_t per = (M[s] + ctx->nranks - 1) / ctx->nranks;
    const int64_t a = std::min<int64_t>(M[s], per * ctx->rank);
    const int64_t b = std::min<int64_t>(M[s], per * (ctx->rank + 1));
    base[s] = a;
    off[s + 1] = off[s] + (b - a);
    xoff[s + 1] = xoff[s] + (b - a) * model->meta[s].d;
    best_std[s] = NAN;  // the fitted incumbent (resolved on the device)
  }
  gpbo_status st = ensure_stage(ctx, (size_t)xoff[S] * 4 + 16);
  if (st) return st;
  float *X = (float *)ctx->stage_d;
  // H5 on a side stream: the generator needs only the space and (for the dedup) the model's
  // training rows, ready after the Gram pre-pass -- so it runs on the SMs the (one-CTA per
  // search) fit leaves idle, and the scoring waits for both
  if (!ctx->gen_stream) {
    CK(cudaStreamCreateWithFlags(&ctx->gen_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->gen_ev, cudaEventDisableTiming));
  }
  if (ctx->xready_ev) CK(cudaStreamWaitEvent(ctx->gen_stream, ctx->xready_ev, 0));
  for (int s = 0; s < S; ++s) {
    const SearchMeta &q = model->meta[s];
    CK(gpbo::launch_gen(gpbo::space_dev(spaces[s]), seed, (uint32_t)s, (uint32_t)iteration,
                        base[s], off[s + 1] - off[s], X + xoff[s],
                        dedup ? model->X32 + q.x_off : nullptr, q.n, ctx->gen_stream));
    ctx->launches += 1;
  }
  CK(cudaEventRecord(ctx->gen_ev, ctx->gen_stream));
  CK(cudaStreamWaitEvent(ctx->stream, ctx->gen_ev, 0));
  std::vector<float> eiv(S);
  st = argmax_tail(ctx, model, X, off.data(), base.data(), best_std.data(), idx, eiv.data());
  if (st) return st;
  int64_t po = 0;
  for (int s = 0; s < S; ++s) {
    const gpbo::SpaceView &v = gpbo::space_host(spaces[s]);
    if (ei) ei[s] = eiv[s];
    if (x_raw) {
      if (idx[s] >= 0) {
        std::vector<float> enc(v.d);
        std::vector<double> vals(v.P);
        gpbo::sample_candidate_host(v, seed, (uint32_t)s, (uint32_t)iteration,
                                    (uint32_t)idx[s], enc.data(), vals.data());
        for (int i = 0; i < v.P; ++i) {
          const int k = v.kind[i];
          double r = vals[i];
          if (k == GPBO_P_REAL) r = v.lo[i] + (v.hi[i] - v.lo[i]) * vals[i];
          else if (k == GPBO_P_INT) r = v.lo[i] + vals[i];
          else if (k == GPBO_P_ORDINAL) r = v.values[v.val_off[i] + (int)vals[i]];
          else if (k == GPBO_P_FIXED) r = v.lo[i];
          x_raw[po + i] = r;
        }
      } else {
        for (int i = 0; i < v.P; ++i) x_raw[po + i] = NAN;
      }
    }
    po += v.P;
  }
  return GPBO_OK;
}

}  // extern "C"
