// lat_stsbar.cu — cost of a CTA barrier preceded by S 128-bit shared stores from one lane per
// warp (the LU panel's candidate-row publish), S = 0, 1, 4, 8, 16, 32; 128 / 256 / 512 threads.
#include <cstdio>
template <int S>
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ __align__(16) double sh[16 * 64 * 2 + 64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double x = 1.0 + tid * 1e-6;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (lane == (i & 31)) {
      double2* d = reinterpret_cast<double2*>(sh + ((i & 1) * 16 + warp) * 64);
#pragma unroll
      for (int c = 0; c < S; ++c) d[c] = make_double2(x, x + c);
    }
    __syncthreads();
    x = sh[((i & 1) * 16 + (lane & 15)) * 64] * 0.5 + 0.5;
  }
  long long t1 = clock64();
  if (!tid) cyc[0] = t1 - t0;
  out[tid] = x;
}
template <int S>
void run(double* o, long long* c, int nt) {
  const int n = 1000;
  k<S><<<1, nt>>>(o, c, n); cudaDeviceSynchronize();
  k<S><<<1, nt>>>(o, c, n); cudaDeviceSynchronize();
  printf("threads %d  sts128 per warp %2d : %.1f cycles per round\n", nt, S, c[0] / (double)n);
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 8 * 8);
  for (int nt : {128, 256, 512}) { run<0>(o, c, nt); run<1>(o, c, nt); run<4>(o, c, nt); run<8>(o, c, nt); run<16>(o, c, nt); run<32>(o, c, nt); }
  return 0;
}
