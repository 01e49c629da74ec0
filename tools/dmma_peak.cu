// FP64 pipe peak microbenchmark for sm_100a (B200).
// Measures register-resident DMMA (mma.sync.m8n8k4.f64) and DFMA throughput so that
// the roofline denominator for the FP64 tile kernels is a measured number, not a
// datasheet figure (SURVEY §8(d) "Peak denominator").
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak dmma_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int NACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5 + 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 0.999999;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 123.456) out[0] = s;
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int iters = 20000;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"", prop.name, sms, prop.major, prop.minor);
  // DMMA: each mma.m8n8k4 = 8*8*4 FMA = 512 flop per warp instruction.
  int thr_list[] = {128, 256, 512};
  for (int ti = 0; ti < 3; ++ti) {
    int thr = thr_list[ti];
    for (int ctas_per_sm = 1; ctas_per_sm <= 2; ++ctas_per_sm) {
      int grid = sms * ctas_per_sm;
      dmma_loop<8><<<grid, thr>>>(out, 100, 1.0);
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        dmma_loop<8><<<grid, thr>>>(out, iters, 1.0);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
      }
      double flops = (double)grid * (thr / 32) * iters * 8 * 512.0;
      printf(", \"dmma_tflops_t%d_c%d\": %.3f", thr, ctas_per_sm, flops / (best * 1e-3) / 1e12);
    }
  }
  for (int ti = 0; ti < 3; ++ti) {
    int thr = thr_list[ti];
    int grid = sms * 2;
    dfma_loop<8><<<grid, thr>>>(out, 100, 1.0);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      dfma_loop<8><<<grid, thr>>>(out, iters * 4, 1.0);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    double flops = (double)grid * thr * iters * 4 * 8 * 2.0;
    printf(", \"dfma_tflops_t%d\": %.3f", thr, flops / (best * 1e-3) / 1e12);
  }
  // sustained DMMA: back-to-back for ~3 s
  {
    int grid = sms, thr = 256;
    CK(cudaEventRecord(e0));
    int n = 0;
    float ms = 0;
    while (ms < 3000.f) {
      dmma_loop<8><<<grid, thr>>>(out, iters, 1.0);
      ++n;
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
    }
    double flops = (double)n * grid * (thr / 32) * iters * 8 * 512.0;
    printf(", \"dmma_tflops_sustained\": %.3f, \"sustained_s\": %.2f", flops / (ms * 1e-3) / 1e12, ms * 1e-3);
  }
  printf("}\n");
  return 0;
}
