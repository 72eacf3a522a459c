// tcgen05.mma rate (M = 128, K = 16, fp16 -> fp32, A from TMEM or SMEM) while other warps load
// from / store to TMEM (the scoring kernel's K* / drain traffic): is the tensor pipe slowed by
// TMEM or shared-memory contention?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2403_08131_b200/csrc -o mma_contention mma_contention.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_prims.cuh"

using namespace gpbo;

// mode bits: 1 = A from TMEM (else SMEM), 2 = loader warps do tcgen05.ld, 4 = they do tcgen05.st,
// 8 = they do shared-memory loads (128-bit, conflict-free)
__global__ void __launch_bounds__(512, 1) bench(int N, int reps, int mode, int rb, long long *out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char *sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0;
  if (threadIdx.x == 0) { tc::mbar_init(tc::smem_u32(&bar), 1); tc::fence_mbar_init(); stop = 0; }
  tc::fence_proxy_async();
  if (warp == 0) tc::tmem_alloc(tc::smem_u32(&slot), 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = slot;
  if (warp == 0) {
    const uint32_t H64 = tc::sdesc_hi((uint32_t)rb);
    const uint32_t blo = tc::sdesc_lo(tc::smem_u32(sm));
    const uint32_t alo = tc::sdesc_lo(tc::smem_u32(sm + 32768));
    const uint32_t idn = tc::idesc_f16((uint32_t)N);
    const long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t dt = tb + ((mode & 64) ? 256u : 0u);
      if (mode & 1) tc::mma_f16_ts(dt, tb + 384, blo, H64, idn, 1u);
      else tc::mma_f16_split(dt, alo, H64, blo, H64, idn, (mode & 128) ? 1u : 0u);
    }
    tc::mma_commit_warp(tc::smem_u32(&bar));
    tc::mbar_wait(tc::smem_u32(&bar), 0);
    const long long c1 = clock64();
    if (lane == 0) { out[0] = c1 - c0; stop = 1; }
  } else if (warp >= 4 && (mode & 16)) {
    // waiting warps: exit at once (no traffic at all)
  } else if (warp >= 4 && (mode & 32)) {
    // waiting warps spin on an mbarrier phase that completes when the MMA loop is done
    tc::mbar_wait(tc::smem_u32(&bar), 0);
  } else if (warp >= 4) {
    const uint32_t ta = tb + ((uint32_t)(32 * (warp & 3)) << 16) + 256 + 32 * ((warp >> 2) & 3);
    long long n = 0;
    uint32_t acc = 0;
    while (!stop) {
      if (mode & 2) {
        uint32_t r[32];
        tc::tmem_ld32(ta, r);
        tc::tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 32; q += 4) acc += r[q];
      }
      if (mode & 4) {
        uint32_t r[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) r[q] = acc + q;
        tc::tmem_st16(ta, r);
        tc::tmem_wait_st();
      }
      if (mode & 8) {
        const uint4 v = reinterpret_cast<const uint4 *>(sm)[(threadIdx.x + 512 * (n & 7)) & 4095];
        acc += v.x ^ v.w;
      }
      ++n;
    }
    if (lane == 0) atomicAdd((unsigned long long *)&out[1], (unsigned long long)n);
    if (acc == 0xdeadbeef) out[2] = acc;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tb, 512);
}

int main() {
  long long *d, h[3];
  cudaMalloc(&d, 24);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const int reps = 2000;
  for (int rb : {64, 128})
  for (int N : {32, 64}) {
    for (int mode : {16, 16 + 64, 16 + 128, 16 + 64 + 128}) {
     for (int thr : {128, 512}) {
      cudaMemset(d, 0, 24);
      bench<<<1, thr, 80 * 1024>>>(N, reps, mode, rb, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
      printf("rb=%3d N=%3d A=%s %s traffic=%s%s%s: %.1f cyc/MMA (floor %d), other-warp iterations %lld %s\n", rb, N,
             (mode & 1) ? "tmem" : "smem", (mode & 16) ? "others-exit" : (mode & 32) ? "others-mbar-wait" : "others-spin-lds", (mode & 2) ? "ld " : "", (mode & 4) ? "st " : "",
             (mode & 8) ? "lds " : "", (double)h[0] / reps, 128 * N / 256, h[1],
             e == cudaSuccess ? "" : cudaGetErrorString(e));
      printf("   (threads %d, D col %d, accumulate %d)\n", thr, (mode & 64) ? 256 : 0, (mode & 128) ? 1 : 0);
     }
    }
  }
  return 0;
}
