// tcgen05 scoring path: envelope, operand-image geometry, launchers (see score_tc.cu).
#pragma once
#include "gpbo_internal.cuh"

namespace gpbo {
constexpr int kTcTile = 128;
// Fills the tcgen05 geometry fields of m (n16, kb, npan, image offsets, tc_ok) from n, d.
void tc_fill_geometry(SearchMeta &m);
bool tc_supported(const SearchMeta &m);
int64_t tc_image_bytes(const SearchMeta &m);
cudaError_t launch_pack_tc(const SearchMeta *meta_d, int S, const double *Linv64,
                           const double *Xs64, const double *alpha64, const float *ls32,
                           unsigned char *img, cudaStream_t stream);
cudaError_t launch_score_tc(const ScoreLaunch &p, const SearchMeta *meta_h, int S,
                            int total_tiles, int num_sms, cudaStream_t stream);
}  // namespace gpbo
