// lat_micro.cu — dependent-chain latencies on one warp: DFMA, DADD, FP64 sqrt, FP64 div,
// 64-bit SHFL, shared-memory load, and the cost of a 512-thread __syncthreads.
#include <cstdio>
__global__ void k(double* out, long long* cyc, int n) {
  double x = 1.0 + threadIdx.x * 1e-6, y = 0.999999;
  long long t0, t1;
  __shared__ double sh[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = i * 1e-3;
  __syncthreads();
  if (threadIdx.x < 32) {
    t0 = clock64(); for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9); t1 = clock64(); if (!threadIdx.x) cyc[0] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < n; ++i) x = x + y; t1 = clock64(); if (!threadIdx.x) cyc[1] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < n; ++i) x = sqrt(x) + 1.0; t1 = clock64(); if (!threadIdx.x) cyc[2] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < n; ++i) x = 2.0 / x + 0.5; t1 = clock64(); if (!threadIdx.x) cyc[3] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * y; t1 = clock64(); if (!threadIdx.x) cyc[4] = t1 - t0;
    int idx = threadIdx.x;
    t0 = clock64(); for (int i = 0; i < n; ++i) { x = sh[idx] * y; idx = ((int)x & 1) + threadIdx.x; } t1 = clock64(); if (!threadIdx.x) cyc[5] = t1 - t0;
  }
  __syncthreads();
  t0 = clock64(); for (int i = 0; i < n; ++i) __syncthreads(); t1 = clock64(); if (!threadIdx.x) cyc[6] = t1 - t0;
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 512 * 8); cudaMallocManaged(&c, 8 * 8);
  const int n = 1000;
  k<<<1, 512>>>(o, c, n); cudaDeviceSynchronize();
  k<<<1, 512>>>(o, c, n); cudaDeviceSynchronize();
  printf("{\"dfma\": %.1f, \"dadd\": %.1f, \"sqrt+add\": %.1f, \"div+add\": %.1f, \"shfl64+mul\": %.1f, \"lds+mul+cvt\": %.1f, \"syncthreads512\": %.1f}\n",
         c[0] / (double)n, c[1] / (double)n, c[2] / (double)n, c[3] / (double)n, c[4] / (double)n, c[5] / (double)n, c[6] / (double)n);
  return 0;
}
