// lupanel_bench.cu — cycles per column of the LU slab panel (tf::lu_panel<MI, TS>) on one
// CTA with the slab in shared memory (round-2 ablations: publish of the pivot row ~350-550,
// rank-1 update ~120-600 cycles per column of 840-2000).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/lupanel tools/lupanel_bench.cu
#include <cstdio>
#include "../paper_0709_1272_b200/csrc/tf_kernels.cuh"
using namespace tf;
#ifndef LUX_NAME
#define LUX_NAME "lu_panel"
#endif
template <int MI, bool TS>
__global__ void __launch_bounds__(TF_THREADS, 1) k(double* out, long long* cyc, int* piv, int reps) {
  extern __shared__ __align__(16) double sm[];
  const int b = 128 * MI, ldp = b + 1;
  double* P = sm;
  double* UL = P + 32 * ldp;
  double* sm2 = UL + 32 * ULD;
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < 32 * ldp; e += TF_THREADS) {
      unsigned h = (unsigned)(e * 2654435761u + r * 40503u);
      h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
      P[e] = (double)(h % 20001) / 10000.0 - 1.0;
    }
    for (int e = threadIdx.x; e < 32 * ULD; e += TF_THREADS) UL[e] = (e % (ULD + 1) == 0) ? 0.9 : 0.01;
    __syncthreads();
    long long t0 = clock64();
    lu_panel<MI, TS>(P, ldp, TS ? 0 : 0, b, UL, piv, sm2, 0);
    long long t1 = clock64();
    tot += t1 - t0;
  }
  if (threadIdx.x == 0) cyc[0] = tot;
  out[threadIdx.x] = P[threadIdx.x];
}
template <int MI, bool TS>
void run(double* o, long long* c, int* pv) {
  const int reps = 20;
  cudaFuncSetAttribute(k<MI, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_DOUBLES * 8);
  k<MI, TS><<<1, TF_THREADS, SMEM_DOUBLES * 8>>>(o, c, pv, 2);
  cudaDeviceSynchronize();
  k<MI, TS><<<1, TF_THREADS, SMEM_DOUBLES * 8>>>(o, c, pv, reps);
  cudaDeviceSynchronize();
  printf("%s b=%d ts=%d cycles/column %.0f\n", LUX_NAME, 128 * MI, (int)TS, c[0] / (double)reps / 32);
}
int main() {
  double* o; long long* c; int* pv;
  cudaMalloc(&o, 512 * 8); cudaMallocManaged(&c, 8); cudaMalloc(&pv, 64 * 4);
  run<1, false>(o, c, pv); run<2, false>(o, c, pv); run<4, false>(o, c, pv);
  run<1, true>(o, c, pv); run<2, true>(o, c, pv); run<4, true>(o, c, pv);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
