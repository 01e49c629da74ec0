// shfl_tput.cu — SM-wide throughput of 64-bit warp shuffles (broadcast from one lane) vs
// one-lane 128-bit shared stores + warp-wide 128-bit broadcast loads, 16 warps of one CTA.
#include <cstdio>
__global__ void k(double* out, long long* cyc, int n, int src) {
  __shared__ __align__(16) double sh[16 * 64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double p[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) p[i] = lane + i * 0.5;
  double acc = 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc += __shfl_sync(0xffffffffu, p[i], (src + it) & 31);
  }
  __syncthreads();
  long long t1 = clock64();
  for (int it = 0; it < n; ++it) {
    if (lane == ((src + it) & 31)) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) *reinterpret_cast<double2*>(sh + warp * 64 + i) = make_double2(p[i], p[i + 1]);
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 16; i += 2) { const double2 v = *reinterpret_cast<const double2*>(sh + warp * 64 + i); acc += v.x + v.y; }
    __syncwarp();
  }
  __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
  out[threadIdx.x] = acc;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 512 * 8); cudaMallocManaged(&c, 16);
  const int n = 200;
  k<<<1, 512>>>(o, c, n, 3); cudaDeviceSynchronize();
  k<<<1, 512>>>(o, c, n, 3); cudaDeviceSynchronize();
  printf("16 warps, 16 doubles from one lane per warp per round: shfl %.0f cycles/round, sts+lds %.0f cycles/round\n",
         c[0] / (double)n, c[1] / (double)n);
  return 0;
}
