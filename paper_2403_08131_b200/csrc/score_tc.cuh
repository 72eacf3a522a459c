// tcgen05 scoring path: envelope, operand-image size, launchers (see score_tc.cu).
#pragma once
#include "gpbo_internal.cuh"

namespace gpbo {
constexpr int kTcTile = 128;
bool tc_supported(const SearchMeta &m);
int64_t tc_image_bytes(const SearchMeta &m);
cudaError_t launch_pack_tc(const SearchMeta *meta_d, int S, const double *Linv64,
                           const float *Xs32, const double *alpha64, unsigned char *img,
                           cudaStream_t stream);
cudaError_t launch_score_tc(const ScoreLaunch &p, int total_tiles, int dmax, int nmax,
                            int num_sms, cudaStream_t stream);
}  // namespace gpbo
