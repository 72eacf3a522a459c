// TMEM load throughput and MUFU throughput on one SM (design input for the scoring kernel's
// K* / drain warps): tcgen05.ld.32x32b.x32 per warp in a loop, W warps, k loads in flight
// before tcgen05.wait::ld; MUFU sqrt + ex2 per element.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2403_08131_b200/csrc -o tmem_micro tmem_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_prims.cuh"

using namespace gpbo;

template <int kInFlight>
__global__ void tmem_ld_bench(float *out, long long *cyc, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc(tc::smem_u32(&slot), 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = slot + ((uint32_t)(32 * (warp & 3)) << 16);
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[kInFlight][32];
#pragma unroll
    for (int k = 0; k < kInFlight; ++k)
      tc::tmem_ld32(tb + (uint32_t)(((i * kInFlight + k) * 32 + 32 * (warp >> 2)) & 511), r[k]);
    tc::tmem_wait_ld();
#pragma unroll
    for (int k = 0; k < kInFlight; ++k)
#pragma unroll
      for (int q = 0; q < 32; q += 8) acc += __uint_as_float(r[k][q]);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = acc;
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(slot, 512);
}

__global__ void mufu_bench(float *out, long long *cyc, int iters) {
  float x[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) x[q] = 1.0f + 1e-3f * (threadIdx.x + q);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      float s, e;
      asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(x[q]));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-s));
      x[q] = e + 1.0f;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  float a = 0.f;
  for (int q = 0; q < 16; ++q) a += x[q];
  out[threadIdx.x] = a;
}

int main() {
  float *out;
  long long *cyc, h;
  cudaMalloc(&out, 4096 * sizeof(float));
  cudaMalloc(&cyc, 8);
  const int iters = 4096;
  for (int w : {4, 8, 16, 32}) {
    for (int k = 1; k <= 4; k *= 2) {
      if (k == 1) tmem_ld_bench<1><<<1, 32 * w>>>(out, cyc, iters);
      if (k == 2) tmem_ld_bench<2><<<1, 32 * w>>>(out, cyc, iters);
      if (k == 4) tmem_ld_bench<4><<<1, 32 * w>>>(out, cyc, iters);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)iters * k * w * 32 * 32 * 4;
      printf("tmem ld x32: %2d warps, %d in flight: %.1f B/clk/SM (%.1f cyc per warp-load)\n", w, k,
             bytes / h, (double)h / (iters * k) );
    }
  }
  for (int w : {4, 8, 16, 32}) {
    mufu_bench<<<1, 32 * w>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops = 2.0 * iters * 16 * w * 32;
    printf("MUFU sqrt+ex2: %2d warps: %.2f MUFU ops/clk/SM\n", w, ops / h);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
