// FP64 / shared-memory / barrier microbenchmarks for the fit kernel's design (one CTA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_micro fp64_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dfma(double *out, long long *cyc, int iters) {
  double a = out[0], b = out[1], c = out[2];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[3] = a; }
}
__global__ void lat_sqrtdiv(double *out, long long *cyc, int iters) {
  double a = out[0] + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { double s = sqrt(a); a = 1.0 / s + 2.0; }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[3] = a; }
}
__global__ void lat_rsqrt(double *out, long long *cyc, int iters) {
  double a = out[0] + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = rsqrt(a) + 2.0; }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[3] = a; }
}
__global__ void thr_dfma(double *out, long long *cyc, int iters) {
  double a0 = out[0] + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = out[1], c = out[2];
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[4 + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void thr_ffma(float *out, long long *cyc, int iters) {
  float a0 = out[0] + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float b = out[1], c = out[2];
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
    a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[4 + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void lat_lds(double *out, long long *cyc, int iters) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
  __syncthreads();
  int p = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = idx[p];
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[3] = p; }
}
__global__ void bar_cost(double *out, long long *cyc, int iters) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void dmma_lat(double *out, long long *cyc, int iters) {
  double d0 = out[0], d1 = out[1], a = out[2], b = out[3];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[8 + threadIdx.x] = d0 + d1;
}
__global__ void dmma_thr(double *out, long long *cyc, int iters) {
  double d[8];
  for (int j = 0; j < 8; ++j) d[j] = out[j];
  const double a = out[2], b = out[3];
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[2 * j]), "+d"(d[2 * j + 1]) : "d"(a), "d"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  double s = 0; for (int j = 0; j < 8; ++j) s += d[j];
  out[8 + threadIdx.x] = s;
}

int main() {
  double *d; long long *c; float *f;
  cudaMalloc(&d, 8 * 2048); cudaMalloc(&c, 64); cudaMalloc(&f, 4 * 2048);
  double h[3] = {1.0000001, 0.9999999, 1e-9};
  cudaMemcpy(d, h, 24, cudaMemcpyHostToDevice);
  float hf[3] = {1.0001f, 0.9999f, 1e-6f};
  cudaMemcpy(f, hf, 12, cudaMemcpyHostToDevice);
  long long r;
  const int it = 4096;
  lat_dfma<<<1, 32>>>(d, c, it); lat_dfma<<<1, 32>>>(d, c, it); cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", r / (4.0 * it));
  lat_sqrtdiv<<<1, 32>>>(d, c, it); lat_sqrtdiv<<<1, 32>>>(d, c, it); cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost);
  printf("sqrt + div + add chain: %.1f cycles\n", r / (double)it);
  lat_rsqrt<<<1, 32>>>(d, c, it); lat_rsqrt<<<1, 32>>>(d, c, it); cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost);
  printf("rsqrt + add chain: %.1f cycles\n", r / (double)it);
  for (int nt : {128, 256, 512, 1024}) {
    thr_dfma<<<1, nt>>>(d, c, it); thr_dfma<<<1, nt>>>(d, c, it); cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA throughput, %4d threads: %.1f FMA/clk/SM\n", nt, 8.0 * it * nt / r);
    thr_ffma<<<1, nt>>>(f, c, it); thr_ffma<<<1, nt>>>(f, c, it); cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost);
    printf("FFMA throughput, %4d threads: %.1f FMA/clk/SM\n", nt, 8.0 * it * nt / r);
  }
  lat_lds<<<1, 32>>>(d, c, it); lat_lds<<<1, 32>>>(d, c, it); cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %.1f cycles\n", r / (double)it);
  for (int nt : {32, 256, 512, 1024}) {
    bar_cost<<<1, nt>>>(d, c, it); bar_cost<<<1, nt>>>(d, c, it); cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads, %4d threads: %.1f cycles\n", nt, r / (double)it);
  }
  dmma_lat<<<1, 32>>>(d, c, it); dmma_lat<<<1, 32>>>(d, c, it); cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost);
  printf("DMMA m8n8k4 dependent latency: %.1f cycles\n", r / (double)it);
  for (int nt : {32, 128, 256, 512}) {
    dmma_thr<<<1, nt>>>(d, c, it); dmma_thr<<<1, nt>>>(d, c, it); cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost);
    printf("DMMA throughput, %4d threads: %.1f FMA/clk/SM\n", nt, 4.0 * 256 * it * (nt / 32) / r);
  }
  return 0;
}
