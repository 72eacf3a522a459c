// H0 (encoding) and H5 (on-device constrained candidate generation) + bo_suggest_batch.
//
// The paper's searches run over expert-constrained spaces ("nstb*nkpb*nspb
// must be less than the total number of allocated cores", "tb*tb_sm ... maximum number of active
// threads per SM"); GPTune "could not even suggest" candidates for the 20-D / 17-D constrained
// joint searches.  Here a candidate is drawn directly from the valid set: each
// constrained block's valid value tuples are enumerated by the caller and one is drawn
// uniformly, free parameters are drawn independently -- no rejection loop.
//
// Counter-based generator: Philox4x32-10, key = (seed lo, seed hi);
// word u (free parameters in declaration order -- fixed ones draw nothing --, then blocks) of global candidate i of search s
// at iteration t = output[u % 4] of Philox(ctr = (i, s, t, u / 4)).  Real: u = (w >> 8) 2^-24;
// K values: index (u64(w >> 8) K) >> 24; block with T tuples: tuple (u64(w >> 8) T) >> 24.
// Encoding (H0, reading R8): real/int (v - lo)/(hi - lo), ordinal rank/(K-1),
// categorical one-hot; float64 then one rounding to float32.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "gpbo_internal.cuh"
#include "space_internal.cuh"

namespace gpbo {

__host__ __device__ inline void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += W0; k1 += W1; }
    const uint64_t p0 = (uint64_t)M0 * c[0];
    const uint64_t p1 = (uint64_t)M1 * c[2];
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0; c[1] = (uint32_t)p1; c[2] = n2; c[3] = (uint32_t)p0;
  }
}

// Draws candidate `idx` and writes its encoding (enc[d]) and, optionally, per-parameter value
// indices / real fractions (vals[P]: index for discrete parameters, u for real ones).
__host__ __device__ inline void sample_candidate(const SpaceView &sp, uint64_t seed, uint32_t search,
                                                 uint32_t iter, uint32_t idx, float *enc,
                                                 double *vals) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  uint32_t word[4];
  int have = -1;
  auto get = [&](int u) -> uint32_t {
    if ((u >> 2) != have) {
      have = u >> 2;
      word[0] = idx; word[1] = search; word[2] = iter; word[3] = (uint32_t)have;
      philox4x32_10(word, k0, k1);
    }
    return word[u & 3];
  };
  auto put = [&](int i, double v) {  // v: u (real) or value index (discrete)
    if (vals) vals[i] = v;
    const int kind = sp.kind[i], col = sp.col[i], K = sp.nv[i];
    if (kind == kReal) {
      enc[col] = (float)v;
    } else if (kind == kCategorical) {
      for (int k = 0; k < K; ++k) enc[col + k] = (k == (int)v) ? 1.f : 0.f;
    } else {
      enc[col] = K > 1 ? (float)(v / (double)(K - 1)) : 0.f;
    }
  };
  for (int f = 0; f < sp.nfree; ++f) {
    const int i = sp.free_list[f];
    const uint32_t w8 = get(f) >> 8;
    if (sp.kind[i] == kReal) put(i, (double)w8 * (1.0 / 16777216.0));
    else put(i, (double)(((uint64_t)w8 * (uint64_t)sp.nv[i]) >> 24));
  }
  for (int b = 0; b < sp.nblocks; ++b) {
    const uint32_t w8 = get(sp.nfree + b) >> 8;
    const int T = sp.tuple_count[b];
    const int bs = sp.block_off[b + 1] - sp.block_off[b];
    const int t = (int)(((uint64_t)w8 * (uint64_t)T) >> 24);
    const int32_t *tp = sp.tuples + sp.tuple_elem_off[b] + (int64_t)t * bs;
    for (int j = 0; j < bs; ++j) put(sp.block_params[sp.block_off[b] + j], (double)tp[j]);
  }
}

namespace {

constexpr int kGenThreads = 128;
constexpr int kHashSlots = 1024;  // >= 2 GPBO_MAX_N: open addressing stays short

// 64-bit hash of an encoded row (FNV-1a style over the columns' bits, then a final mix); +0 and
// -0 hash alike (they compare equal).  Training rows and candidates are hashed the same way.
__device__ __forceinline__ uint64_t row_hash(const float *r, int d) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (int c = 0; c < d; ++c) {
    const float v = r[c] == 0.f ? 0.f : r[c];
    h = (h ^ __float_as_uint(v)) * 0x100000001B3ull;
  }
  h ^= h >> 29;
  h *= 0xBF58476D1CE4E5B9ull;
  return h ^ (h >> 32);
}

// One candidate per thread, 128 per CTA: drawn into a shared-memory tile (row stride d | 1:
// conflict-free), deduplicated against the training rows through a shared-memory hash table of
// their encodings (reading R14: a candidate equal to an observed configuration is masked with
// NaN; equality is exact, the hash only selects which rows to compare), then written to HBM as
// one contiguous, coalesced block.
__global__ void __launch_bounds__(kGenThreads)
gen_kernel(const SpaceView sp_g, uint64_t seed, uint32_t search, uint32_t iter, int64_t first,
           int64_t count, float *out, const float *__restrict__ Xtrain, int n) {
  extern __shared__ float tile[];
  __shared__ unsigned long long hkey[kHashSlots];
  __shared__ int hrow[kHashSlots];
  // the per-parameter tables (P <= GPBO_MAX_D) in shared memory: sample_candidate reads them
  // once per parameter and candidate
  __shared__ int32_t s_kind[GPBO_MAX_D], s_nv[GPBO_MAX_D], s_col[GPBO_MAX_D], s_free[GPBO_MAX_D];
  const int tid = threadIdx.x;
  for (int i = tid; i < sp_g.P; i += kGenThreads) {
    s_kind[i] = sp_g.kind[i]; s_nv[i] = sp_g.nv[i]; s_col[i] = sp_g.col[i];
  }
  for (int i = tid; i < sp_g.nfree; i += kGenThreads) s_free[i] = sp_g.free_list[i];
  SpaceView sp = sp_g;
  sp.kind = s_kind; sp.nv = s_nv; sp.col = s_col; sp.free_list = s_free;
  __syncthreads();
  const int d = sp.d, ld = d | 1;
  if (Xtrain) {
    for (int e = tid; e < kHashSlots; e += kGenThreads) { hkey[e] = 0ull; hrow[e] = -1; }
    __syncthreads();
    for (int j = tid; j < n; j += kGenThreads) {
      const uint64_t h = row_hash(Xtrain + (size_t)j * d, d) | 1ull;  // 0 marks an empty slot
      for (int sl = (int)(h & (kHashSlots - 1));; sl = (sl + 1) & (kHashSlots - 1)) {
        if (atomicCAS(&hkey[sl], 0ull, (unsigned long long)h) == 0ull) { hrow[sl] = j; break; }
      }
    }
    __syncthreads();
  }
  float *enc = tile + tid * ld;
  const int64_t ntile = (count + kGenThreads - 1) / kGenThreads;
  for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x) {  // persistent: one table build per CTA
    const int64_t i0 = t * kGenThreads;
    const int cnt = (int)min((int64_t)kGenThreads, count - i0);
    __syncthreads();  // the previous tile's rows are written out
    if (tid < cnt) {
      sample_candidate(sp, seed, search, iter, (uint32_t)(first + i0 + tid), enc, nullptr);
      if (Xtrain) {
        const uint64_t h = row_hash(enc, d) | 1ull;
        bool dup = false;
        for (int sl = (int)(h & (kHashSlots - 1)); !dup && hkey[sl] != 0ull;
             sl = (sl + 1) & (kHashSlots - 1)) {
          if (hkey[sl] != h) continue;
          const float *xr = Xtrain + (size_t)hrow[sl] * d;
          bool eq = true;
          for (int c = 0; c < d && eq; ++c) eq = xr[c] == enc[c];
          dup = eq;
        }
        if (dup) enc[0] = NAN;
      }
    }
    __syncthreads();
    // coalesced write-out: element e = r d + c of the tile, (r, c) advanced incrementally
    float *dst = out + i0 * d;
    const int step_r = kGenThreads / d, step_c = kGenThreads - step_r * d;
    int r = tid / d, c = tid - r * d;
    for (int e = tid; e < cnt * d; e += kGenThreads) {
      dst[e] = tile[r * ld + c];
      r += step_r;
      c += step_c;
      if (c >= d) { c -= d; ++r; }
    }
  }
}

}  // namespace

cudaError_t launch_gen(const SpaceView &sp_dev, uint64_t seed, uint32_t search, uint32_t iter,
                       int64_t first, int64_t count, float *out, const float *Xtrain, int n,
                       cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  if (n > kHashSlots / 2) return cudaErrorInvalidValue;
  const size_t smem = (size_t)kGenThreads * (sp_dev.d | 1) * sizeof(float);
  static std::atomic<int> sms_of[64];  // SM count per device (0 = not yet queried)
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64) {
    sms = sms_of[dev].load(std::memory_order_relaxed);
    if (sms == 0) {
      if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
      sms_of[dev].store(sms, std::memory_order_relaxed);
    }
  }
  const int64_t tiles = (count + kGenThreads - 1) / kGenThreads;
  gen_kernel<<<(unsigned)std::min<int64_t>(tiles, (int64_t)std::max(sms, 1) * 8), kGenThreads, smem, st>>>(
      sp_dev, seed, search, iter, first, count, out, Xtrain, n);
  return cudaGetLastError();
}

void sample_candidate_host(const SpaceView &sp, uint64_t seed, uint32_t search, uint32_t iter,
                           uint32_t idx, float *enc, double *vals) {
  sample_candidate(sp, seed, search, iter, idx, enc, vals);
}

}  // namespace gpbo

// ------------------------------------------------------------------ space objects (host side)
using gpbo::SpaceView;

struct gpbo_space {
  int device = 0;
  SpaceView host{}, dev{};
  std::vector<int32_t> ints;
  std::vector<double> dbls;
  void *dblob = nullptr;
};

namespace {

// Lays the description out as one int array + one double array; `base_*` rebase the pointers.
void build_view(SpaceView &v, const int32_t *ib, const double *db, const std::vector<int> &ioff,
                const std::vector<int> &doff, int P, int d, int nfree, int nblocks) {
  v.P = P; v.d = d; v.nfree = nfree; v.nblocks = nblocks;
  v.kind = ib + ioff[0]; v.nv = ib + ioff[1]; v.col = ib + ioff[2]; v.free_list = ib + ioff[3];
  v.block_off = ib + ioff[4]; v.block_params = ib + ioff[5]; v.tuple_count = ib + ioff[6];
  v.tuple_elem_off = ib + ioff[7]; v.tuples = ib + ioff[8]; v.val_off = ib + ioff[9];
  v.lo = db + doff[0]; v.hi = db + doff[1]; v.values = db + doff[2];
}

}  // namespace

extern "C" {

gpbo_status gpbo_space_create(gpbo_ctx *ctx, const gpbo_space_desc *s, gpbo_space **out) {
  if (!ctx || !s || !out) return GPBO_EINVAL;
  *out = nullptr;
  const int P = s->P;
  if (P < 1 || !s->kind || !s->nvals || !s->lo || !s->hi || (s->nblocks > 0 &&
      (!s->block_off || !s->block_params || !s->tuple_off || !s->tuples)))
    return GPBO_EINVAL;
  std::vector<int32_t> kind(s->kind, s->kind + P), nv(P), col(P);
  std::vector<int> inblock(P, 0);
  int d = 0;
  for (int i = 0; i < P; ++i) {
    const int k = kind[i];
    if (k < 0 || k > 4) return GPBO_EINVAL;
    if (k == GPBO_P_FIXED) {  // no column, no draw: its value is lo
      if (!std::isfinite(s->lo[i])) return GPBO_EINVAL;
      nv[i] = 0;
      col[i] = d;
      continue;
    }
    if (k == GPBO_P_REAL) {
      if (!(s->hi[i] > s->lo[i])) return GPBO_EINVAL;
      nv[i] = 0;
    } else if (k == GPBO_P_INT) {
      nv[i] = (int32_t)std::llround(s->hi[i] - s->lo[i]) + 1;
    } else {
      nv[i] = s->nvals[i];
    }
    if (k != GPBO_P_REAL && (nv[i] < 1 || nv[i] > (1 << 24))) return GPBO_EINVAL;
    if (k == GPBO_P_ORDINAL && (!s->values || !s->val_off)) return GPBO_EINVAL;
    col[i] = d;
    d += k == GPBO_P_CATEGORICAL ? nv[i] : 1;
  }
  if (d > GPBO_MAX_D) return GPBO_EINVAL;
  const int nb = s->nblocks;
  std::vector<int32_t> boff(nb + 1, 0), bpar, tcnt(nb), toff(nb + 1, 0), tup;
  for (int b = 0; b < nb; ++b) {
    const int a = s->block_off[b], e = s->block_off[b + 1];
    if (e <= a) return GPBO_EINVAL;
    for (int j = a; j < e; ++j) {
      const int i = s->block_params[j];
      if (i < 0 || i >= P || kind[i] == GPBO_P_REAL || kind[i] == GPBO_P_FIXED || inblock[i])
        return GPBO_EINVAL;
      inblock[i] = 1;
      bpar.push_back(i);
    }
    boff[b + 1] = (int32_t)bpar.size();
    const int T = s->tuple_off[b + 1] - s->tuple_off[b];
    if (T < 1) return GPBO_ESAMPLING;  // an empty valid set cannot be sampled
    tcnt[b] = T;
  }
  // copy tuples: tuple_off counts tuples; element offset = sum over previous blocks T_b * bs_b
  {
    int64_t eoff = 0;
    tup.clear();
    for (int b = 0; b < nb; ++b) {
      const int bs = boff[b + 1] - boff[b];
      const int T = tcnt[b];
      toff[b] = (int32_t)tup.size();
      for (int64_t e = 0; e < (int64_t)T * bs; ++e) {
        const int v = s->tuples[eoff + e];
        const int i = bpar[boff[b] + (int)(e % bs)];
        if (v < 0 || v >= nv[i]) return GPBO_EINVAL;
        tup.push_back(v);
      }
      eoff += (int64_t)T * bs;
    }
  }
  std::vector<int32_t> freel;
  for (int i = 0; i < P; ++i)
    if (!inblock[i] && kind[i] != GPBO_P_FIXED) freel.push_back(i);
  std::vector<int32_t> voff(P, 0);
  std::vector<double> vals;
  for (int i = 0; i < P; ++i) {
    voff[i] = (int32_t)vals.size();
    if (kind[i] == GPBO_P_ORDINAL)
      for (int k = 0; k < nv[i]; ++k) vals.push_back(s->values[s->val_off[i] + k]);
  }
  gpbo_space *sp = new gpbo_space();
  sp->device = 0;
  std::vector<int> ioff, doff;
  auto addi = [&](const std::vector<int32_t> &v) {
    ioff.push_back((int)sp->ints.size());
    sp->ints.insert(sp->ints.end(), v.begin(), v.end());
    sp->ints.push_back(0);  // never empty
  };
  auto addd = [&](const std::vector<double> &v) {
    doff.push_back((int)sp->dbls.size());
    sp->dbls.insert(sp->dbls.end(), v.begin(), v.end());
    sp->dbls.push_back(0.0);
  };
  addi(kind); addi(nv); addi(col); addi(freel); addi(boff); addi(bpar); addi(tcnt); addi(toff);
  addi(tup); addi(voff);
  addd(std::vector<double>(s->lo, s->lo + P));
  addd(std::vector<double>(s->hi, s->hi + P));
  addd(vals);
  build_view(sp->host, sp->ints.data(), sp->dbls.data(), ioff, doff, P, d, (int)freel.size(), nb);
  const size_t db = sp->dbls.size() * 8, ib = sp->ints.size() * 4;
  if (cudaMalloc(&sp->dblob, db + ib) != cudaSuccess) { delete sp; return GPBO_ENOMEM; }
  cudaMemcpy(sp->dblob, sp->dbls.data(), db, cudaMemcpyHostToDevice);
  cudaMemcpy((char *)sp->dblob + db, sp->ints.data(), ib, cudaMemcpyHostToDevice);
  build_view(sp->dev, (const int32_t *)((char *)sp->dblob + db), (const double *)sp->dblob, ioff,
             doff, P, d, (int)freel.size(), nb);
  *out = sp;
  return GPBO_OK;
}

void gpbo_space_free(gpbo_space *sp) {
  if (!sp) return;
  if (sp->dblob) cudaFree(sp->dblob);
  delete sp;
}

int32_t gpbo_space_dim(const gpbo_space *sp) { return sp ? sp->host.d : -1; }

gpbo_status gpbo_space_encode(const gpbo_space *sp, const double *raw, float *enc) {
  if (!sp || !raw || !enc) return GPBO_EINVAL;
  const SpaceView &v = sp->host;
  for (int i = 0; i < v.P; ++i) {
    const int k = v.kind[i], col = v.col[i], K = v.nv[i];
    const double x = raw[i];
    if (!std::isfinite(x)) return GPBO_EINVAL;
    if (k == GPBO_P_FIXED) continue;  // no encoded column
    if (k == GPBO_P_REAL || k == GPBO_P_INT) {
      enc[col] = (float)((x - v.lo[i]) / (v.hi[i] - v.lo[i]));
    } else if (k == GPBO_P_ORDINAL) {
      int r = -1;
      for (int q = 0; q < K; ++q)
        if (v.values[v.val_off[i] + q] == x) r = q;
      if (r < 0) return GPBO_EINVAL;
      enc[col] = K > 1 ? (float)((double)r / (double)(K - 1)) : 0.f;
    } else {
      const int r = (int)std::llround(x);
      if (r < 0 || r >= K || (double)r != x) return GPBO_EINVAL;
      for (int q = 0; q < K; ++q) enc[col + q] = q == r ? 1.f : 0.f;
    }
  }
  return GPBO_OK;
}

}  // extern "C"

namespace gpbo {
const SpaceView &space_dev(const gpbo_space *sp) { return sp->dev; }
const SpaceView &space_host(const gpbo_space *sp) { return sp->host; }
}  // namespace gpbo
