// DMMA issue-pattern microbenchmark: the GEMM engine's warp-tile pattern (MI x NI
// accumulators, a[h][i] / b[h][j] operands varying per DMMA) with register-resident
// operands (no shared-memory loads), to separate the DMMA pipe's own limit for that
// pattern from the engine's operand staging.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/dmma_pattern tools/dmma_pattern.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MI, int NI>
__global__ void __launch_bounds__(512, 1) pat(double* out, int iters, double seed) {
  double acc[MI][NI][2];
  double a[2][MI], b[2][NI];
#pragma unroll
  for (int i = 0; i < MI; ++i) { a[0][i] = seed + i + threadIdx.x; a[1][i] = seed - i; }
#pragma unroll
  for (int j = 0; j < NI; ++j) { b[0][j] = seed * j; b[1][j] = seed + 2 * j; }
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]) : "d"(a[h][i]), "d"(b[h][j]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 123.456) out[0] = s;
}

template <int MI, int NI>
void run(const char* name, int threads, int sms, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  pat<MI, NI><<<sms, threads>>>(out, 10, 1.0);
  cudaEventRecord(e0);
  pat<MI, NI><<<sms, threads>>>(out, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 512.0 * 2 * MI * NI * iters * (threads / 32) * (double)sms;
  printf("{\"pattern\": \"%s\", \"threads\": %d, \"tflops\": %.3f}\n", name, threads, fl / (ms * 1e-3) / 1e12);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  run<4, 4>("32x32 warp tile (16 acc)", 512, sms, out);
  run<4, 4>("32x32 warp tile (16 acc)", 128, sms, out);
  run<2, 4>("16x32 (8 acc)", 512, sms, out);
  run<4, 2>("32x16 (8 acc)", 512, sms, out);
  run<8, 4>("64x32 (32 acc)", 256, sms, out);
  run<1, 1>("1 acc", 512, sms, out);
  return 0;
}
