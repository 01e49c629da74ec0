// div_check.cu — tf::div_rcp(x, d, tf::rcp_newton(d)) against the compiler's x / d, bitwise,
// over random (x, d) pairs: signs, exponents spread over [-1000, 1000] (both paths of the
// guard), plus N(0,1)-like magnitudes (the LU panel's values) and special values.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/div_check tools/div_check.cu
//   ./build/div_check [rounds]   -> {"pairs": N, "mismatches": M}
#include <cstdio>
#include <cstdlib>
#include "../paper_0709_1272_b200/csrc/tf_common.cuh"

__device__ unsigned long long mix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ double gen(unsigned long long h, int mode) {
  const unsigned long long m = h & 0xfffffffffffffull, s = (h >> 63) << 63;
  int e;
  if (mode == 0) e = 1023 + (int)((h >> 52) % 2001) - 1000;          // wide exponents
  else if (mode == 1) e = 1023 + (int)((h >> 52) % 41) - 20;          // the panel's range
  else e = (int)((h >> 52) % 2048);                                   // everything incl. inf/nan/denormals
  const unsigned long long bits = s | ((unsigned long long)e << 52) | m;
  return __longlong_as_double((long long)bits);
}
__global__ void k(unsigned long long seed, unsigned long long* bad, unsigned long long n) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long h1 = mix(seed ^ (2 * i)), h2 = mix(seed ^ (2 * i + 1));
    const int mode = (int)(i % 3);
    const double x = gen(h1, mode), d = gen(h2, mode);
    const double a = x / d, b = tf::div_rcp(x, d, tf::rcp_newton(d));
    const bool same = (__double_as_longlong(a) == __double_as_longlong(b)) || (a != a && b != b);
    if (!same) atomicAdd(bad, 1ull);
  }
}
int main(int argc, char** argv) {
  const int rounds = argc > 1 ? atoi(argv[1]) : 16;
  unsigned long long* bad;
  cudaMallocManaged(&bad, 8);
  *bad = 0;
  const unsigned long long n = 1ull << 28;
  for (int r = 0; r < rounds; ++r) k<<<148 * 8, 256>>>(0x1234567ull + r * 0x10001ull, bad, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"pairs\": %llu, \"mismatches\": %llu, \"cuda\": \"%s\"}\n", n * rounds, *bad, cudaGetErrorString(e));
  return (*bad == 0 && e == cudaSuccess) ? 0 : 1;
}
