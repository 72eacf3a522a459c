// Self-test of the tcgen05 building blocks (operand swizzle layouts, UMMA descriptors, k-advance
// inside a swizzle row, B-operand row offsets, TMEM allocation / loads, MMA commit): one CTA
// computes D[128 x N] = A[128 x K] * B[N x K]^T in fp16 -> fp32 exactly as the scoring kernel
// issues its MMAs.  Exposed as the test hook gpbo_tc_selftest (include/gpbo.h).
#include <cuda_fp16.h>

#include "gpbo_internal.cuh"
#include "tc_prims.cuh"

namespace gpbo {
namespace {

__global__ void __launch_bounds__(128, 1)
tc_selftest_kernel(const __half *A, const __half *B, float *D, int N, int K, int row_bytes,
                   int b_row_off, int timing, long long *cycles) {
  extern __shared__ unsigned char sm_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kpb = row_bytes / 2;  // fp16 elements per swizzle row
  const int nkb = K / kpb;
  const int Nb = N + b_row_off;
  unsigned char *sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
  unsigned char *As = sm;
  unsigned char *Bs = sm + ((128 * K * 2 + 1023) & ~1023);
  // stage operands in the K-major swizzled layout
  for (int e = tid; e < 128 * K; e += 128) {
    const int r = e / K, k = e % K, kb = k / kpb, kk = k % kpb;
    *reinterpret_cast<__half *>(As + kb * 128 * row_bytes + tc::sw_offset(r, kk * 2, row_bytes)) =
        A[e];
  }
  for (int e = tid; e < Nb * K; e += 128) {
    const int r = e / K, k = e % K, kb = k / kpb, kk = k % kpb;
    const __half v = r >= b_row_off ? B[(r - b_row_off) * K + k] : __float2half(1e4f);
    *reinterpret_cast<__half *>(Bs + kb * Nb * row_bytes + tc::sw_offset(r, kk * 2, row_bytes)) =
        v;
  }
  tc::fence_proxy_async();
  if (tid == 0) { tc::mbar_init(tc::smem_u32(&bar), 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc(tc::smem_u32(&tmem_base), 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (timing < 0) {
    // A operand from TMEM: thread = row, 16 fp16 of one k step packed in 8 columns (k = 2c, 2c+1)
    const int row = warp * 32 + lane;
    for (int s = 0; s < K / 16; ++s) {
      uint32_t r[8];
      for (int c = 0; c < 8; ++c) {
        const __half lo = A[row * K + 16 * s + 2 * c], hi = A[row * K + 16 * s + 2 * c + 1];
        r[c] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
      }
      tc::tmem_st8(tbase + ((uint32_t)(warp * 32) << 16) + 256 + 8 * s, r);
    }
    tc::tmem_wait_st();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (warp == 0) {
      const uint32_t b0 = tc::smem_u32(Bs);
      const uint32_t H = tc::sdesc_hi(row_bytes);
      const uint32_t idesc = tc::idesc_f16(N);
      int first = 1;
      for (int kb = 0; kb < nkb; ++kb)
        for (int s = 0; s < kpb / 16; ++s) {
          const uint32_t blo = tc::sdesc_lo(b0 + kb * Nb * row_bytes +
                                            (b_row_off / 8) * 8 * row_bytes + s * 32);
          tc::mma_f16_ts(tbase, tbase + 256 + 8 * (kb * (kpb / 16) + s), blo, H, idesc,
                         first ? 0u : 1u);
          first = 0;
        }
      tc::mma_commit_warp(tc::smem_u32(&bar));
    }
  } else if (tid == 0) {
    const uint32_t a0 = tc::smem_u32(As), b0 = tc::smem_u32(Bs);
    const uint32_t idesc = tc::idesc_f16(N);
    int first = 1;
    for (int kb = 0; kb < nkb; ++kb)
      for (int s = 0; s < kpb / 16; ++s) {
        const uint64_t ad = tc::make_sdesc(a0 + kb * 128 * row_bytes + s * 32, row_bytes);
        const uint64_t bd = tc::make_sdesc(
            b0 + kb * Nb * row_bytes + (b_row_off / 8) * 8 * row_bytes + s * 32, row_bytes);
        tc::mma_f16(tbase, ad, bd, idesc, first ? 0u : 1u);
        first = 0;
      }
    tc::mma_commit(tc::smem_u32(&bar));
  }
  tc::mbar_wait(tc::smem_u32(&bar), 0);
  if (timing > 0 && warp == 0) {
    // issue-rate microbenchmark: `timing` repetitions of the same accumulate MMA by the whole
    // warp (elected lane), clock64 after issue and after completion
    const uint32_t H = tc::sdesc_hi(row_bytes);
    const uint32_t alo = tc::sdesc_lo(tc::smem_u32(As)), blo = tc::sdesc_lo(tc::smem_u32(Bs));
    const uint32_t idesc = tc::idesc_f16(N);
    const long long c0 = clock64();
    for (int r = 0; r < timing; ++r) tc::mma_f16_split(tbase + 256, alo, H, blo, H, idesc, 1u);
    const long long c1 = clock64();
    tc::mma_commit_warp(tc::smem_u32(&bar));
    tc::mbar_wait(tc::smem_u32(&bar), 1);
    const long long c2 = clock64();
    if (lane == 0) { cycles[0] = c1 - c0; cycles[1] = c2 - c0; }
  }
  __syncthreads();
  tc::tc_fence_after();
  for (int c = 0; c < N; c += 8) {
    uint32_t r[8];
    tc::tmem_ld8(tbase + ((uint32_t)(warp * 32) << 16) + c, r);
    tc::tmem_wait_ld();
    for (int q = 0; q < 8; ++q) D[(warp * 32 + lane) * N + c + q] = __uint_as_float(r[q]);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

}  // namespace
}  // namespace gpbo

extern "C" gpbo_status gpbo_tc_bench(const void *A, const void *B, float *D, int N, int K,
                                     int row_bytes, int b_row_off, int reps, long long *cycles);

extern "C" gpbo_status gpbo_tc_selftest(const void *A, const void *B, float *D, int N, int K,
                                        int row_bytes, int b_row_off) {
  return gpbo_tc_bench(A, B, D, N, K, row_bytes, b_row_off, 0, nullptr);
}

extern "C" gpbo_status gpbo_tc_bench(const void *A, const void *B, float *D, int N, int K,
                                     int row_bytes, int b_row_off, int reps, long long *cycles) {
  if (!A || !B || !D || N < 16 || N > 256 || N % 16 || K < 16 ||
      (row_bytes != 32 && row_bytes != 64 && row_bytes != 128) || K % (row_bytes / 2) ||
      b_row_off < 0 || b_row_off % 8)
    return GPBO_EINVAL;
  const int smem = ((128 * K * 2 + 1023) & ~1023) + (N + b_row_off) * K * 2 + 1024;
  if (smem > 200 * 1024) return GPBO_EINVAL;
  if (cudaFuncSetAttribute(gpbo::tc_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           smem) != cudaSuccess)
    return GPBO_ECUDA;
  long long *cyc = nullptr;
  if (reps > 0 && cudaMalloc(&cyc, 16) != cudaSuccess) return GPBO_ECUDA;
  // reps < 0: A operand staged in TMEM (tcgen05.st) and read by the MMA from TMEM
  gpbo::tc_selftest_kernel<<<1, 128, smem>>>((const __half *)A, (const __half *)B, D, N, K,
                                             row_bytes, b_row_off, reps, cyc);
  if (reps > 0) {
    cudaMemcpy(cycles, cyc, 16, cudaMemcpyDeviceToHost);
    cudaFree(cyc);
  }
  return cudaDeviceSynchronize() == cudaSuccess ? GPBO_OK : GPBO_ECUDA;
}
