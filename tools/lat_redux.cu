// lat_redux.cu — dependent-chain latencies (cycles) of the LU panel's primitives on one warp:
// redux.sync max/min (u32), the 3-redux first-max, FP64 division, LDS.64, STS+BAR+LDS (4 / 16 warps).
#include <cstdio>
#include <climits>
__device__ __forceinline__ void wfm(double v, int idx, double& bv, int& bi) {
  const unsigned hi = (unsigned)__double2hiint(v), lo = (unsigned)__double2loint(v);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  bi = __reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? idx : INT_MAX);
  bv = __hiloint2double((int)mhi, (int)mlo);
}
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double sh[1024];
  __shared__ double xch[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 1024; i += blockDim.x) sh[i] = 1.0 + i * 1e-3;
  __syncthreads();
  double x = 1.0 + tid * 1e-6;
  unsigned u = tid;
  long long t0, t1;
  if (warp == 0) {
    t0 = clock64(); for (int i = 0; i < n; ++i) u = __reduce_max_sync(0xffffffffu, u + lane); t1 = clock64(); if (!tid) cyc[0] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < n; ++i) u = __reduce_min_sync(0xffffffffu, (int)(u + lane)); t1 = clock64(); if (!tid) cyc[1] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < n; ++i) { double bv; int bi; wfm(x, lane, bv, bi); x = bv * 0.999 + bi * 1e-9 + lane * 1e-12; } t1 = clock64(); if (!tid) cyc[2] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < n; ++i) x = 2.0 / x + 0.5; t1 = clock64(); if (!tid) cyc[3] = t1 - t0;
    int idx = lane;
    t0 = clock64(); for (int i = 0; i < n; ++i) { x = sh[idx]; idx = ((int)x & 1) + lane; } t1 = clock64(); if (!tid) cyc[4] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < n; ++i) x = fma(x, 0.999, 1e-9); t1 = clock64(); if (!tid) cyc[5] = t1 - t0;
  }
  __syncthreads();
  // exchange round: every warp writes one value, barrier, every lane reads 16 values' max (one LDS)
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (lane == 0) xch[(i & 1) * 32 + warp] = x;
    __syncthreads();
    x = xch[(i & 1) * 32 + (lane & 15)] * 0.5 + 0.5;
  }
  t1 = clock64(); if (!tid) cyc[6] = t1 - t0;
  out[tid] = x + u;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 8 * 8);
  const int n = 1000;
  for (int nt : {128, 256, 512}) {
    k<<<1, nt>>>(o, c, n); cudaDeviceSynchronize();
    k<<<1, nt>>>(o, c, n); cudaDeviceSynchronize();
    printf("{\"threads\": %d, \"redux_max\": %.1f, \"redux_min\": %.1f, \"first_max3+\": %.1f, \"ddiv+add\": %.1f, \"lds64\": %.1f, \"dfma\": %.1f, \"sts_bar_lds\": %.1f}\n", nt,
           c[0] / (double)n, c[1] / (double)n, c[2] / (double)n, c[3] / (double)n, c[4] / (double)n, c[5] / (double)n, c[6] / (double)n);
  }
  return 0;
}
