// fp64_alu.cu — throughput of non-tensor FP64 FMA (DFMA) and FP64 add on one SM
// (16 warps, 8 independent chains per thread), to size scalar FP64 work in panels.
#include <cstdio>
__global__ void k(double* out, long long* cyc, int n) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double m = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], m, c);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 148 * 512 * 8); cudaMallocManaged(&c, 148 * 8);
  const int n = 4096;
  k<<<148, 512>>>(o, c, n); cudaDeviceSynchronize();
  k<<<148, 512>>>(o, c, n); cudaDeviceSynchronize();
  double fl = 512.0 * 8 * n;  // FMAs per SM
  printf("{\"dfma_per_clk_per_sm\": %.2f}\n", fl / (double)c[0]);
  return 0;
}
