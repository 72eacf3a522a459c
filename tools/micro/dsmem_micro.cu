// DSMEM / cluster-barrier microbenchmark (cluster of 8 CTAs x 384 threads):
//  mode 0: cluster.sync() only
//  mode 1: every thread stores 16 doubles into each of the 8 CTAs (remote push), then sync
//  mode 2: every thread stores 16 doubles locally, sync, then loads 16 doubles from each CTA (pull)
//  mode 3: as 1 but only warp 0 stores (64 doubles x 8 CTAs: the map broadcast)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(384) k(int mode, int iters, long long *out, double *sink) {
  __shared__ double buf[8 * 384 * 2];
  cg::cluster_group cl = cg::this_cluster();
  const int r = cl.block_rank();
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 1 || (mode == 3 && threadIdx.x < 32)) {
      for (int q = 0; q < 8; ++q) {
        double *dst = cl.map_shared_rank(buf, q);
        for (int e = 0; e < (mode == 3 ? 2 : 2); ++e) dst[(r * 384 + threadIdx.x) * 2 + e] = it + e;
      }
    } else if (mode == 2) {
      buf[(r * 384 + threadIdx.x) * 2] = it;
    }
    cl.sync();
    if (mode == 2) {
      for (int q = 0; q < 8; ++q) {
        const double *src = cl.map_shared_rank(buf, q);
        acc += src[(q * 384 + threadIdx.x) * 2];
      }
      cl.sync();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && r == 0) out[mode] = (t1 - t0) / iters;
  if (acc == 12345.0) sink[0] = acc;
}
int main() {
  long long *o; double *s;
  cudaMalloc(&o, 64); cudaMalloc(&s, 8);
  for (int mode = 0; mode < 4; ++mode) {
    k<<<8, 384>>>(mode, 200, o, s);
    cudaDeviceSynchronize();
    long long h[4];
    cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
    printf("mode %d: %lld cycles per iteration (%s)\n", mode, h[mode], cudaGetErrorString(cudaGetLastError()));
  }
}
