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


// F2FP (cvt.rn.f16x2.f32) throughput alone and mixed with MUFU: does the pack share the XU pipe?
template <int kMode>  // 0: F2FP only, 1: MUFU only, 2: both interleaved
__global__ void f2fp_bench(float *out, long long *cyc, int iters) {
  float x[16];
  uint32_t acc = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) x[q] = 1.0f + 1e-3f * (threadIdx.x + q);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 16; q += 2) {
      const float y = x[q + 1];
      if (kMode != 1) {
        uint32_t h;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x[q]), "f"(y));
        acc ^= h;
      }
      float e = 1e-3f;
      if (kMode != 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-y));
      x[q + 1] = fmaf(y, 0.999f, e);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = x[0] + x[15] + (float)acc;
}

int main() {
  float *out;
  long long *cyc, h;
  cudaMalloc(&out, 4096 * sizeof(float));
  cudaMalloc(&cyc, 8);
  const int iters = 4096;
  for (int w : {4, 8, 16}) {
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
  for (int mode = 0; mode < 3; ++mode) {
    if (mode == 0) f2fp_bench<0><<<1, 512>>>(out, cyc, iters);
    if (mode == 1) f2fp_bench<1><<<1, 512>>>(out, cyc, iters);
    if (mode == 2) f2fp_bench<2><<<1, 512>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops = 8.0 * iters * 512;  // per kind
    printf("mode %d (0 F2FP, 1 MUFU, 2 both): %.2f ops of each kind /clk/SM\n", mode, ops / h);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
