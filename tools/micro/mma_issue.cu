// Issue cost of the scoring kernel's variance-MMA loop (one warp, A from TMEM, B from shared
// memory, per 16-wide k step the three fp16x3 products hi.hi, hi.lo, lo.hi with run-time
// descriptors): separate asm statements per MMA (ptxas moves every operand to uniform registers
// per MMA) vs one asm statement per k step (shared operands moved once).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2403_08131_b200/csrc -o mma_issue mma_issue.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_prims.cuh"

using namespace gpbo;

// three products of one k step in one statement: D += A.Bh, D += A.Bl, D += Alo.Bh
__device__ __forceinline__ void mma3_ts(uint32_t d, uint32_t a, uint32_t blo, uint32_t bhi,
                                        uint32_t boff, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 b0, b1;\n\t.reg .b32 t, a2;\n\t"
      "add.u32 t, %2, %4;\n\t"
      "add.u32 a2, %1, 32;\n\t"
      "mov.b64 b0, {%2, %3};\n\t"
      "mov.b64 b1, {t, %3};\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], b0, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], b1, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b0, %5, 1;\n\t}"
      ::"r"(d), "r"(a), "r"(blo), "r"(bhi), "r"(boff), "r"(idesc), "r"(acc)
      : "memory");
}

// one thread issues (no elect.sync / divergence checks per MMA)
__device__ __forceinline__ void mma_ts1(uint32_t d, uint32_t a, uint32_t blo, uint32_t bhi,
                                        uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 db;\n\t"
      "mov.b64 db, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, p;\n\t}"
      ::"r"(d), "r"(a), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit1(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__global__ void __launch_bounds__(128, 1) bench(const int *prm, int reps, int mode, long long *out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char *sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 16 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    tc::mbar_init(tc::smem_u32(&bar), 1);
    tc::mbar_init(tc::smem_u32(&bar2), 1);
    tc::fence_mbar_init();
  }
  tc::fence_proxy_async();
  if (warp == 0) tc::tmem_alloc(tc::smem_u32(&slot), 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = slot;
  if (warp == 0) {
    int n16 = prm[0];  // run-time values, as in the kernel (meta from global memory)
    uint32_t tbase_ = tbase;
    if (mode & 256) {  // make the bases provably warp-uniform (ptxas can keep them in URs)
      n16 = __shfl_sync(0xffffffffu, n16, 0);
      tbase_ = __shfl_sync(0xffffffffu, tbase_, 0);
    }
    const uint32_t tbase = tbase_;
    const int P64 = (n16 + 63) / 64;
    const uint32_t H64 = tc::sdesc_hi(64);
    uint32_t l0 = tc::sdesc_lo(tc::smem_u32(sm));
    if (mode & 256) l0 = __shfl_sync(0xffffffffu, l0, 0);
    const long long c0 = clock64();
    int nmma = 0;
    if (mode & 32) {  // loop-invariant operands (as gpbo_tc_bench): SS or TS
      const uint32_t idn = tc::idesc_f16(32u);
      for (int r = 0; r < reps * 39; ++r) {
        const uint32_t acc = (mode & 64) ? (r > 0 ? 1u : 0u) : 1u;
        if (mode & 1) tc::mma_f16_ts(tbase, tbase + 384u, l0, H64, idn, acc);
        else tc::mma_f16_split(tbase, l0, H64, l0 + (uint32_t)prm[1], H64, idn, acc);
      }
      nmma = reps * 39;
    } else
    for (int r = 0; r < reps; ++r) {
      for (int v_pp = 0; v_pp < P64; ++v_pp) {
        const uint32_t kt = tbase + 384u + 64u * (uint32_t)(r & 1);
#pragma unroll
        for (int sk = 0; sk < 4; ++sk) {
          const int j0 = 64 * v_pp + 16 * sk;
          if (j0 < n16) {
            const int pp = 2 * v_pp + (sk >> 1), h = sk & 1;
            const uint32_t R16 = (uint32_t)(n16 - 32 * pp) * 4u;
            const uint32_t lp = l0 + (uint32_t)(pp * n16 - 16 * pp * (pp - 1)) * 8u;
            // small N keeps the pipe below the issue cost (this measures the issue loop)
            const uint32_t idn = tc::idesc_f16(mode & 2 ? (uint32_t)(n16 - j0) : 32u);
            const uint32_t dt = tbase + (uint32_t)j0;
            const uint32_t ka = kt + 8u * sk;
            const uint32_t lb = lp + 66u * h;
            const uint32_t acc = (v_pp | sk) ? 1u : 0u;
            if (mode & 16) {
              if (lane == 0) {
                mma_ts1(dt, ka, lb, H64, idn, acc);
                mma_ts1(dt, ka, lb + R16, H64, idn, 1u);
                mma_ts1(dt, ka + 32u, lb, H64, idn, 1u);
                if (mode & 4) commit1(tc::smem_u32(&bar2));
              }
              __syncwarp();
            } else if (mode & 1) {
              mma3_ts(dt, ka, lb, H64, R16, idn, acc);
            } else {
              tc::mma_f16_ts(dt, ka, lb, H64, idn, acc);
              tc::mma_f16_ts(dt, ka, lb + R16, H64, idn, 1u);
              tc::mma_f16_ts(dt, ka + 32u, lb, H64, idn, 1u);
            }
            nmma += 3;
            if ((mode & 4) && !(mode & 16)) tc::mma_commit_warp(tc::smem_u32(&bar2));
            if (mode & 8) tc::mma_commit(tc::smem_u32(&bar2));
          }
        }
      }
    }
    tc::mma_commit_warp(tc::smem_u32(&bar));
    tc::mbar_wait(tc::smem_u32(&bar), 0);
    const long long c1 = clock64();
    if (lane == 0) { out[0] = c1 - c0; out[1] = nmma; }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

int main() {
  long long *d, h[2];
  int *prm, hp[2] = {208, 0};
  cudaMalloc(&d, 16);
  cudaMalloc(&prm, 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  const int smem_kb = 120;
  for (int mode : {0, 2, 256, 258, 256 + 4, 256 + 6}) {
    hp[1] = 1024;
    cudaMemcpy(prm, hp, 8, cudaMemcpyHostToDevice);
    printf("mode %d: ", mode);
    bench<<<1, 128, smem_kb * 1024>>>(prm, 200, mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%s%s, N %s: %.1f cyc/MMA over %lld MMAs %s\n", (mode & 32) ? ((mode & 1) ? ((mode & 64) ? "invariant TS, D zeroed first" : "invariant TS") : ((mode & 64) ? "invariant SS, D zeroed first" : "invariant SS")) : (mode & 16) ? "lane 0 issues" : (mode & 1) ? "one asm per k step" : "one asm per MMA", (mode & 4) ? " + commit per k step" : "",
           (mode & 2) ? "= kernel's (n16 - j0)" : "= 32", (double)h[0] / h[1], h[1],
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
