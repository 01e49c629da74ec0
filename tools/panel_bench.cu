// panel_bench.cu — cycles per column of the slab Householder panel (slab_panel<MI>) on one
// CTA with the panel in shared memory; -DEXP_* variants switch parts off to locate cost.
#include <cstdio>
#include "../paper_0709_1272_b200/csrc/tf_kernels.cuh"
using namespace tf;
template <int MI>
__global__ void __launch_bounds__(TF_THREADS, 1) pb_kernel(double* out, long long* cyc, int reps, int ts) {
  extern __shared__ __align__(16) double sm[];
  const int b = 128 * MI, ldp = b + 1;
  double* P = sm;
  double* Rb = P + 32 * ldp;
  double* Ts = Rb + 33 * 32;
  double* sm2 = Ts + 33 * 32;
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < 32 * ldp; e += TF_THREADS) P[e] = 1e-3 * ((e * 2654435761u) % 1000) + (e % (ldp + 1) == 0 ? 1.0 : 0.0);
    for (int e = threadIdx.x; e < 33 * 32; e += TF_THREADS) Rb[e] = (e % 34 == 0) ? 2.0 : 0.01;
    __syncthreads();
    long long t0 = clock64();
    if (ts) slab_panel<MI, true>(P, ldp, 0, Rb, Ts, sm2);
    else slab_panel<MI, false>(P, ldp, 0, Rb, Ts, sm2);
    long long t1 = clock64();
    tot += t1 - t0;
  }
  if (threadIdx.x == 0) cyc[0] = tot;
  out[threadIdx.x] = P[threadIdx.x];
}
int main(int argc, char** argv) {
  double* o; long long* c;
  cudaMalloc(&o, 512 * 8); cudaMallocManaged(&c, 8);
  const int reps = 20;
  cudaFuncSetAttribute(pb_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_DOUBLES * 8);
  cudaFuncSetAttribute(pb_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_DOUBLES * 8);
  for (int ts = 0; ts < 2; ++ts) {
    pb_kernel<2><<<1, TF_THREADS, SMEM_DOUBLES * 8>>>(o, c, reps, ts); cudaDeviceSynchronize();
    printf("b=256 ts=%d cycles/column %.0f\n", ts, c[0] / (double)reps / 32);
    pb_kernel<4><<<1, TF_THREADS, SMEM_DOUBLES * 8>>>(o, c, reps, ts); cudaDeviceSynchronize();
    printf("b=512 ts=%d cycles/column %.0f\n", ts, c[0] / (double)reps / 32);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
