// chol_bench.cu — cycles of the 32x32 diagonal-block Cholesky (tf::chol_diag_block, warp 0)
// on one CTA, SPD input from a fixed pattern; variants below are local experiments.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/chol_bench tools/chol_bench.cu
#include <cstdio>
#include "../paper_0709_1272_b200/csrc/tf_kernels.cuh"
using namespace tf;

// variant: the same algorithm with row j staged in registers of every lane by ONE 32-wide
// shared load per column (lane m reads L[j][m]) and shuffled to lanes as needed
__device__ inline int chol_v1(double* D, int* sflag) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double x[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) x[c] = c <= lane ? D[lane + c * (NB + 1)] : 0.0;
    int fail = -1;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      // all of row j at once (lane m: L[j][m]), then broadcast per m by shuffle
      const double rowj = lane < j ? D[j + lane * (NB + 1)] : 0.0;
      double p[4] = {x[j], 0.0, 0.0, 0.0};
#pragma unroll
      for (int m = 0; m < j; ++m) p[m & 3] -= x[m] * __shfl_sync(0xffffffffu, rowj, m);
      const double sj = (p[0] + p[1]) + (p[2] + p[3]);
      const double d = __shfl_sync(0xffffffffu, sj, j);
      if (!(d > 0.0)) { fail = j; break; }
      const double r = rsqrt(d);
      if (lane == j) { x[j] = d * r; D[j + j * (NB + 1)] = x[j]; D[NB + j * (NB + 1)] = r; }
      else if (lane > j) { x[j] = sj * r; D[lane + j * (NB + 1)] = x[j]; }
      __syncwarp();
    }
    if (lane == 0) *sflag = fail;
  }
  __syncthreads();
  return *sflag;
}

// variant: no early exit (a failing column is recorded and the arithmetic runs on), one
// predicated select + one predicated store per column instead of two divergent branches
__device__ inline int chol_v2(double* D, int* sflag) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double x[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) x[c] = c <= lane ? D[lane + c * (NB + 1)] : 0.0;
    int fail = -1;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      double p[4] = {x[j], 0.0, 0.0, 0.0};
#pragma unroll
      for (int m = 0; m < j; ++m) p[m & 3] -= x[m] * D[j + m * (NB + 1)];
      const double sj = (p[0] + p[1]) + (p[2] + p[3]);
      const double d = __shfl_sync(0xffffffffu, sj, j);
      if (!(d > 0.0) && fail < 0) fail = j;
      const double r = rsqrt(d);
      const double v = (lane == j ? d : sj) * r;
      if (lane >= j) {
        x[j] = v;
        D[lane + j * (NB + 1)] = v;
      }
      if (lane == j) D[NB + j * (NB + 1)] = r;
      __syncwarp();
    }
    if (lane == 0) *sflag = fail;
  }
  __syncthreads();
  return *sflag;
}


// v3: right-looking; lane i holds row i; after column j every lane applies the rank-1 update
// to its remaining entries with L[c][j] read back from shared memory (broadcast loads), and
// the next pivot d_{j+1} = x_{j+1}[j+1] - L[j+1][j]^2 is formed by lane j+1 and shuffled
// (the critical path per column: shuffle, rsqrt, one multiply, one FMA)
__device__ inline int chol_v3(double* D, int* sflag) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double x[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) x[c] = D[lane + c * (NB + 1)];
    int fail = -1;
    double d = __shfl_sync(0xffffffffu, x[0], 0);
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      if (!(d > 0.0) && fail < 0) fail = j;
      const double r = rsqrt(d);
      const double l = (lane == j ? d : x[j]) * r;
      if (lane >= j) D[lane + j * (NB + 1)] = l;
      if (lane == j) D[NB + j * (NB + 1)] = r;
      if (j + 1 < NB) {
        d = __shfl_sync(0xffffffffu, x[j + 1] - l * l, j + 1);
        __syncwarp();
#pragma unroll
        for (int c = j + 1; c < NB; ++c) x[c] -= l * D[c + j * (NB + 1)];
      }
    }
    if (lane == 0) *sflag = fail;
  }
  __syncthreads();
  return *sflag;
}

template <int V>
__global__ void __launch_bounds__(TF_THREADS, 1) k(double* out, long long* cyc, int reps) {
  __shared__ double D[(NB + 1) * NB];
  __shared__ int sflag;
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < NB * NB; e += TF_THREADS) {
      const int i = e % NB, j = e / NB;
      D[i + j * (NB + 1)] = (i == j) ? 64.0 + r : 1.0 / (1 + i + j);
    }
    __syncthreads();
    const long long t0 = clock64();
    const int f = V == 0 ? chol_diag_block(D, NB, &sflag) : V == 1 ? chol_v1(D, &sflag) : V == 2 ? chol_v2(D, &sflag) : chol_v3(D, &sflag);
    const long long t1 = clock64();
    tot += t1 - t0;
    if (f >= 0 && threadIdx.x == 0) out[1] = f;
  }
  if (threadIdx.x == 0) cyc[V] = tot;
  for (int e = threadIdx.x; e < NB * (NB + 1); e += TF_THREADS) out[8 + V * NB * (NB + 1) + e] = D[e];
}
int main() {
  double* o; long long* c;
  cudaMallocManaged(&o, 8 * (8 + 4 * NB * (NB + 1))); cudaMallocManaged(&c, 64);
  const int reps = 50;
  for (int it = 0; it < 2; ++it) {
    k<0><<<1, TF_THREADS>>>(o, c, reps); k<1><<<1, TF_THREADS>>>(o, c, reps); k<2><<<1, TF_THREADS>>>(o, c, reps);
    k<3><<<1, TF_THREADS>>>(o, c, reps);
    cudaDeviceSynchronize();
  }
  printf("chol_diag_block: %.0f cycles/column; v1 (row via shuffles): %.0f; v2 (no exit, predicated): %.0f\n",
         c[0] / (double)reps / NB, c[1] / (double)reps / NB, c[2] / (double)reps / NB);
  double md = 0, mref = 0;
  for (int j = 0; j < NB; ++j)
    for (int i = j; i <= NB; ++i) {  // lower triangle and the reciprocal padding row
      const double a = o[8 + i + j * (NB + 1)], b = o[8 + 3 * NB * (NB + 1) + i + j * (NB + 1)];
      md = fmax(md, fabs(a - b)); mref = fmax(mref, fabs(a));
    }
  printf("v3 (right-looking): %.0f cycles/column; max |v3 - v0| = %.3g (max |v0| %.3g)\n", c[3] / (double)reps / NB, md, mref);
  return 0;
}
