// Latency of tcgen05.ld (+ wait::ld) and tcgen05.st (+ wait::st) issued by one warp while another
// warp keeps the tensor pipe busy with MMAs into other TMEM columns (the scoring kernel's K*
// warps load distances / store K* while variance MMAs run): are TMEM accesses queued behind
// in-flight MMAs?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2403_08131_b200/csrc -o tmem_ld_lat tmem_ld_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_prims.cuh"

using namespace gpbo;

__global__ void __launch_bounds__(128, 1) bench(int N, int nmma, int mma_on, int a_tmem, int fence_mode, long long *out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char *sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 32 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0;
  if (threadIdx.x == 0) { tc::mbar_init(tc::smem_u32(&bar), 1); tc::fence_mbar_init(); done = 0; }
  tc::fence_proxy_async();
  if (warp == 0) tc::tmem_alloc(tc::smem_u32(&slot), 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = slot;
  if (warp == 0) {
    if (mma_on) {
      const uint32_t H = tc::sdesc_hi(32);
      const uint32_t blo = tc::sdesc_lo(tc::smem_u32(sm)), alo = tc::sdesc_lo(tc::smem_u32(sm + 16384));
      const uint32_t idn = tc::idesc_f16((uint32_t)N);
      for (int r = 0; r < nmma; ++r) {
        if (a_tmem) tc::mma_f16_ts(tb, tb + 448u, blo, H, idn, 1u);
        else tc::mma_f16_split(tb, alo, H, blo, H, idn, 1u);
      }
      tc::mma_commit_warp(tc::smem_u32(&bar));
      tc::mbar_wait(tc::smem_u32(&bar), 0);
    } else {
      const long long c0 = clock64();
      while (clock64() - c0 < 200000) {}
    }
    if (lane == 0) done = 1;
  } else if (warp == 1 || warp == 2) {
    // warp 1: loads from columns [256, 288) (lanes 32..63); warp 2: stores to [320, 336)
    const uint32_t ta = tb + ((uint32_t)(32 * warp) << 16);
    long long tot = 0, mx = 0, n = 0;
    uint32_t acc = 0;
    while (!done && n < 4000) {
      const long long c0 = clock64();
      if (fence_mode & 1) tc::tc_fence_after();
      if (fence_mode & 2) tc::tc_fence_before();
      if (warp == 1) {
        uint32_t r[32];
        tc::tmem_ld32(ta + 256u, r);
        tc::tmem_wait_ld();
        acc += r[0] ^ r[31];
      } else {
        uint32_t r[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) r[q] = acc + q;
        tc::tmem_st16(ta + 320u, r);
        tc::tmem_wait_st();
      }
      const long long dt = clock64() - c0;
      tot += dt;
      mx = dt > mx ? dt : mx;
      ++n;
      const long long c1 = clock64();
      while (clock64() - c1 < 200) {}
    }
    if (lane == 0) { out[2 * (warp - 1)] = tot / (n ? n : 1); out[2 * (warp - 1) + 1] = mx; out[4 + warp - 1] = n; }
    if (acc == 0xdeadbeefu) out[7] = acc;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tb, 512);
}

int main() {
  long long *d, h[8];
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int fm : {0, 1, 2})
  for (int mma_on : {0, 1})
    for (int a_tmem : {1})
      for (int N : {224}) {
        printf("fence %s: ", fm == 1 ? "after_thread_sync before ld" : fm == 2 ? "before_thread_sync before ld" : "none");
        cudaMemset(d, 0, 64);
        bench<<<1, 128, 40 * 1024>>>(N, 2000, mma_on, a_tmem, fm, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
        printf("MMAs %s (A %s, N=%3d): tcgen05.ld x32+wait avg %lld max %lld cyc (%lld samples); "
               "tcgen05.st x16+wait avg %lld max %lld (%lld) %s\n", mma_on ? "running" : "idle   ",
               a_tmem ? "tmem" : "smem", N, h[0], h[1], h[4], h[2], h[3], h[5],
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
