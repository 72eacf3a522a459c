// CTA-pair (cta_group::2) tcgen05 MMA check: D[256 x N] = A[256 x 16] B[N x 16]^T with A from
// TMEM (each CTA its 128 rows, as the scoring kernel's K* operand) or from shared memory, B split
// by rows across the pair (CTA r holds B rows [r N/2, (r+1) N/2) at the same shared offset),
// D in each CTA's TMEM (its 128 rows x N).  Verifies the operand split and times the issue rate.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2403_08131_b200/csrc -o pair_mma pair_mma.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "tc_prims.cuh"

using namespace gpbo;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t idesc_f16_m256(uint32_t N) {
  return (1u << 4) | ((N >> 3) << 17) | ((256u >> 4) << 24);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
pair_kernel(const __half *A, const __half *B, float *D, int N, int a_tmem, int reps, long long *cyc) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char *sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t rank = cluster_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char *As = sm;           // 128 rows x 32 B (SW32, K = 16)
  unsigned char *Bs = sm + 4096;    // N/2 rows x 32 B
  const int Nh = N / 2;
  for (int e = tid; e < 128 * 16; e += 128) {
    const int r = e / 16, k = e % 16;
    *reinterpret_cast<__half *>(As + tc::sw_offset(r, k * 2, 32)) = A[(128 * rank + r) * 16 + k];
  }
  for (int e = tid; e < Nh * 16; e += 128) {
    const int r = e / 16, k = e % 16;
    *reinterpret_cast<__half *>(Bs + tc::sw_offset(r, k * 2, 32)) = B[(Nh * rank + r) * 16 + k];
  }
  tc::fence_proxy_async();
  if (tid == 0) { tc::mbar_init(tc::smem_u32(&bar), 1); tc::fence_mbar_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = slot;
  // A in TMEM: lane = row, 8 columns of packed fp16 pairs at column 384
  {
    const int row = warp * 32 + lane;
    uint32_t r[8];
    for (int c = 0; c < 8; ++c) {
      const __half lo = A[(128 * rank + row) * 16 + 2 * c], hi = A[(128 * rank + row) * 16 + 2 * c + 1];
      r[c] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
    }
    tc::tmem_st8(tb + ((uint32_t)(warp * 32) << 16) + 384, r);
    tc::tmem_wait_st();
  }
  tc::tc_fence_before();
  cluster_sync();  // both CTAs' operands are in place (and both barriers initialised)
  tc::tc_fence_after();
  if (rank == 0 && warp == 0) {
    const uint32_t H32 = tc::sdesc_hi(32);
    const uint32_t alo = tc::sdesc_lo(tc::smem_u32(As)), blo = tc::sdesc_lo(tc::smem_u32(Bs));
    const uint32_t idn = idesc_f16_m256((uint32_t)N);
    const long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t acc = r > 0 ? 1u : 0u;
      if (a_tmem) {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t.reg .b64 db;\n\t"
            "mov.b64 db, {%2, %3};\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %5, 0;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], db, %4, p;\n\t}"
            ::"r"(tb), "r"(tb + 384u), "r"(blo), "r"(H32), "r"(idn), "r"(acc) : "memory");
      } else {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\t"
            "mov.b64 da, {%1, %2};\n\t"
            "mov.b64 db, {%3, %2};\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %5, 0;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %4, p;\n\t}"
            ::"r"(tb), "r"(alo), "r"(H32), "r"(blo), "r"(idn), "r"(acc) : "memory");
      }
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
        ::"r"(tc::smem_u32(&bar)), "h"((unsigned short)3) : "memory");
    tc::mbar_wait(tc::smem_u32(&bar), 0);
    const long long c1 = clock64();
    if (lane == 0) cyc[0] = c1 - c0;
  }
  tc::mbar_wait(tc::smem_u32(&bar), 0);
  tc::tc_fence_after();
  for (int c = 0; c < N; c += 8) {
    uint32_t r[8];
    tc::tmem_ld8(tb + ((uint32_t)(warp * 32) << 16) + c, r);
    tc::tmem_wait_ld();
    for (int q = 0; q < 8; ++q) D[(128 * rank + warp * 32 + lane) * N + c + q] = __uint_as_float(r[q]);
  }
  tc::tc_fence_before();
  cluster_sync();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512) : "memory");
}

int main() {
  for (int a_tmem = 0; a_tmem < 2; ++a_tmem)
  for (int N : {32, 64, 128, 224, 256}) {
    const int M = 256, K = 16;
    __half *hA = (__half *)malloc(M * K * 2), *hB = (__half *)malloc(N * K * 2);
    float *hD = (float *)malloc(M * N * 4);
    for (int i = 0; i < M * K; ++i) hA[i] = __float2half((float)((i * 7) % 13) - 6.f);
    for (int i = 0; i < N * K; ++i) hB[i] = __float2half((float)((i * 5) % 11) - 5.f);
    __half *dA, *dB; float *dD; long long *dc, hc[1];
    cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dc, 8);
    cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, N * K * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
    // correctness: reps = 1
    pair_kernel<<<2, 128, 32 * 1024>>>(dA, dB, dD, N, a_tmem, 1, dc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)__half2float(hA[i * K + k]) * __half2float(hB[j * K + k]);
        maxerr = fmax(maxerr, fabs(ref - hD[i * N + j]));
      }
    const int reps = 2000;
    pair_kernel<<<2, 128, 32 * 1024>>>(dA, dB, dD, N, a_tmem, reps, dc);
    cudaError_t e2 = cudaDeviceSynchronize();
    cudaMemcpy(hc, dc, 8, cudaMemcpyDeviceToHost);
    printf("A from %s N=%3d: max |err| %.3g  %.1f cyc/MMA (M = 256)  %s %s\n", a_tmem ? "TMEM" : "SMEM", N,
           maxerr, (double)hc[0] / reps, cudaGetErrorString(e), cudaGetErrorString(e2));
  }
  return 0;
}
