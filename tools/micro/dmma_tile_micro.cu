// Microbenchmark of the fit's trailing-update work item (fit.cu "quad"): per 8 x 8 tile one
// 16-byte accumulator load, two B-fragment loads, two DMMA m8n8k4, one 16-byte store.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_tile_micro dmma_tile_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int kMode>
__global__ void quads(double *out, long long *cyc, int nq) {
  extern __shared__ __align__(16) double sm[];
  double *W = sm, *G = sm + 300 * 64;  // 300 tiles + G (8 x 216)
  for (int i = threadIdx.x; i < 300 * 64 + 8 * 216; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gid = lane >> 2, tig = lane & 3;
  const int gs = 216;
  long long t0 = clock64();
  double acc = 0.0;
  for (int it = 0; it < nq; ++it) {
    const int R = (warp * 7 + it * 3) % 24 + 1, C0 = (it * 5 + warp) % (R > 3 ? R - 3 : 1);
    const int cnt = kMode == 2 ? 4 : 4 - (it & 1);
    const int i = 8 * R + gid;
    if (kMode == 3) {  // DMMA only (register operands)
      double c0 = acc, c1 = acc, a = 1e-3 * it, b = 2e-3;
#pragma unroll
      for (int q = 0; q < 8; ++q) dmma(c0, c1, a, b);
      acc += c0 + c1;
      continue;
    }
    const double a0 = -G[tig * gs + i], a1 = -G[(4 + tig) * gs + i];
    double *Wt = W + ((R * (R + 1) / 2 + C0) % 290) * 64 + 2 * lane;
    const double *g0 = G + tig * gs + 8 * C0 + gid, *g1 = g0 + 4 * gs;
    if (kMode == 0) {  // serial per tile (the fit's first form)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q < cnt) {
          double2 c = *reinterpret_cast<double2 *>(Wt + 64 * q);
          dmma(c.x, c.y, a0, g0[8 * q]);
          dmma(c.x, c.y, a1, g1[8 * q]);
          *reinterpret_cast<double2 *>(Wt + 64 * q) = c;
        }
      }
    } else {  // staged: all loads, then the DMMAs, then the stores
      double2 c[4];
      double b0[4], b1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < cnt) {
          c[q] = *reinterpret_cast<const double2 *>(Wt + 64 * q);
          b0[q] = g0[8 * q];
          b1[q] = g1[8 * q];
        }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < cnt) dmma(c[q].x, c[q].y, a0, b0[q]);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < cnt) dmma(c[q].x, c[q].y, a1, b1[q]);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < cnt) *reinterpret_cast<double2 *>(Wt + 64 * q) = c[q];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = acc + sm[threadIdx.x];
}

int main() {
  double *d; long long *c;
  cudaMalloc(&d, 8 * 2048); cudaMalloc(&c, 64);
  const int smem = (300 * 64 + 8 * 216) * 8;
  cudaFuncSetAttribute(quads<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(quads<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(quads<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(quads<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int nq = 200;
  for (int nt : {128, 256, 384, 512}) {
    long long r[4];
    for (int mode = 0; mode < 4; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) quads<0><<<1, nt, smem>>>(d, c, nq);
        if (mode == 1) quads<1><<<1, nt, smem>>>(d, c, nq);
        if (mode == 2) quads<2><<<1, nt, smem>>>(d, c, nq);
        if (mode == 3) quads<3><<<1, nt, smem>>>(d, c, nq);
      }
      cudaMemcpy(&r[mode], c, 8, cudaMemcpyDeviceToHost);
    }
    const double tiles = nq * 3.5 * (nt / 32);
    printf("%4d threads: cycles/tile serial %.1f  staged %.1f  staged-full4 %.1f (x4/3.5)  dmma-only(8/quad) %.1f  | DMMA-bound %.1f\n",
           nt, r[0] / tiles, r[1] / tiles, r[2] / (nq * 4.0 * (nt / 32)), r[3] / (nq * 4.0 * (nt / 32)), 2 * 256 / 64.0);
  }
  return 0;
}
