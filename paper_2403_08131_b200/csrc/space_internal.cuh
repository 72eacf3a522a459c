// Search-space view shared by the generator kernel (space.cu) and bo_suggest_batch (api.cu).
#pragma once
#include <cstdint>

#include "gpbo_internal.cuh"

namespace gpbo {

enum { kReal = GPBO_P_REAL, kInt = GPBO_P_INT, kOrdinal = GPBO_P_ORDINAL,
       kCategorical = GPBO_P_CATEGORICAL, kFixed = GPBO_P_FIXED };

struct SpaceView {
  int32_t P, d, nfree, nblocks;
  const int32_t *kind, *nv, *col, *free_list;
  const int32_t *block_off, *block_params, *tuple_count, *tuple_elem_off, *tuples, *val_off;
  const double *lo, *hi, *values;
};

cudaError_t launch_gen(const SpaceView &sp_dev, uint64_t seed, uint32_t search, uint32_t iter,
                       int64_t first, int64_t count, float *out, const float *Xtrain, int n,
                       cudaStream_t st);
void sample_candidate_host(const SpaceView &sp, uint64_t seed, uint32_t search, uint32_t iter,
                           uint32_t idx, float *enc, double *vals);
}  // namespace gpbo

struct gpbo_space;
namespace gpbo {
const SpaceView &space_dev(const gpbo_space *sp);
const SpaceView &space_host(const gpbo_space *sp);
}  // namespace gpbo
