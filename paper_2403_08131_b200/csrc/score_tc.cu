// tcgen05 scoring path -- placeholder until the tensor-core kernel lands.
#include "score_tc.cuh"

namespace gpbo {
bool tc_supported(const SearchMeta &) { return false; }
int64_t tc_image_bytes(const SearchMeta &) { return 0; }
cudaError_t launch_pack_tc(const SearchMeta *, int, const double *, const float *,
                           const double *, unsigned char *, cudaStream_t) {
  return cudaSuccess;
}
cudaError_t launch_score_tc(const ScoreLaunch &, int, int, int, int, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace gpbo
