// dmma_lat.cu — latency of a dependent chain of DMMA.8x8x4 and of shared-memory-fed DMMAs
// (one warp), to size the software pipelining of the small SSRFB / T-phase products.
#include <cstdio>
#include "../paper_0709_1272_b200/csrc/tf_common.cuh"
using namespace tf;
__global__ void lat(double* out, long long* cyc, int n) {
  double c[2] = {0, 0};
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) dmma(c, a, b);
  __syncwarp();
  long long t1 = clock64();
  out[threadIdx.x] = c[0] + c[1];
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // 8 independent chains
  double d[8][2] = {};
  t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(d[k], a, b);
  __syncwarp();
  t1 = clock64();
  double s = 0;
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  out[32 + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 64 * 8); cudaMallocManaged(&c, 16);
  lat<<<1, 32>>>(o, c, 1024);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, c, 1024);
  cudaDeviceSynchronize();
  printf("{\"dmma_dep_chain_cycles\": %.1f, \"dmma_8chains_cycles_per_dmma\": %.2f}\n", c[0] / 1024.0, c[1] / 8192.0);
  return 0;
}
