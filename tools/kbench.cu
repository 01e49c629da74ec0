// kbench.cu — per-kernel throughput microbenchmark for the tile kernels of libtilefact.
// Every CTA runs work items of one kind back to back on its own private tiles (no
// scheduler, no dependencies), so the measured rate is the kernel's steady-state
// per-SM throughput, directly comparable with the trace's per-item numbers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -o build/kbench tools/kbench.cu
//   ./build/kbench <kind> <b> <ib> [ctas_per_sm=1] [reps=4]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
// the same noinline per-variant functions as the persistent kernel (TF_SPLIT_ITEMS), so the
// measured code is the code the scheduler runs
#define TF_SPLIT_ITEMS
#include "../paper_0709_1272_b200/csrc/tf_kernels.cuh"

using namespace tf;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void __launch_bounds__(TF_THREADS, 1)
kb_kernel(int kind, int b, int ib, double* tiles, double* aux, int* ipiv, double* scratch, size_t scr, int reps,
          int shared_ab) {
  extern __shared__ __align__(16) double sm[];
  Ctx cx;
  cx.b = b; cx.ib = ib; cx.scratch = scratch + (size_t)blockIdx.x * scr; cx.info = nullptr; cx.abort_flag = nullptr;
  cx.nopiv = 0;
  const size_t bb = (size_t)b * b;
  double* t0 = tiles + (size_t)blockIdx.x * 3 * bb;
  double* t1 = t0 + bb;
  double* t2 = t1 + bb;
  if (shared_ab) {  // every CTA reads the same two operand tiles (L2-resident), own output tile
    t0 = tiles;
    t1 = tiles + bb;
  }
  double* ax = aux + (size_t)blockIdx.x * ib * b;
  int* pv = ipiv + (size_t)blockIdx.x * b;
  const int nit = items_of(kind, b, ib);
  pipe_init(sm);
  for (int r = 0; r < reps; ++r) {
    const int it = (blockIdx.x + r) % nit;
    if (threadIdx.x == 0) fence_proxy_async_all();
#ifdef KB_KIND
    // single-kind build (nvcc -DKB_KIND=<id>): compiles in a fraction of the time
    if (kind != KB_KIND) continue;
#endif
    switch (kind) {
#if !defined(KB_KIND) || KB_KIND == 0
      case 0: potrf_item(cx, t0, sm); break;
#endif
#if !defined(KB_KIND) || KB_KIND == 1
      case 1: trsm_item(cx, t0, t1, it, sm); break;
#endif
#if !defined(KB_KIND) || KB_KIND == 2
      case 2: syrk_item(cx, t0, t1, it, sm); break;
#endif
#if !defined(KB_KIND) || KB_KIND == 3
      case 3: gemm_item(cx, t0, t1, t2, it, sm); break;
#endif
#if !defined(KB_KIND) || KB_KIND == 4
      case 4: geqrt_item(cx, t0, ax, t2, sm); break;
#endif
#if !defined(KB_KIND) || KB_KIND == 5
      case 5: larfb_item(cx, t0, ax, t1, it, sm); break;
#endif
#if !defined(KB_KIND) || KB_KIND == 6
      case 6: tsqrt_item(cx, t0, t1, ax, sm); break;
#endif
#if !defined(KB_KIND) || KB_KIND == 7
      case 7: ssrfb_item(cx, t0, ax, t1, t2, it, sm); break;
#endif
#if !defined(KB_KIND) || KB_KIND == 8
      case 8: getrf_item(cx, t0, pv, t2, sm); break;
#endif
#if !defined(KB_KIND) || KB_KIND == 9
      case 9: gessm_item(cx, t0, pv, t1, it, sm); break;
#endif
#if !defined(KB_KIND) || KB_KIND == 10
      case 10: tstrf_item(cx, t0, t1, ax, pv, sm); break;
#endif
#if !defined(KB_KIND) || KB_KIND == 11
      case 11: ssssm_item(cx, t0, ax, pv, t1, t2, it, sm); break;
#endif
    }
    __syncthreads();
  }
}

__global__ void init_kernel(double* x, size_t n, int b, int kind) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    // diagonally dominant, well-scaled values so repeated in-place application stays finite
    const size_t w = e % ((size_t)b * b);
    const int r = (int)(w % b), c = (int)(w / b);
    double v = 1e-3 * (double)((e * 2654435761ull) % 1000) / 1000.0;
    if (r == c) v += (kind == 0) ? 1e6 : 4.0;
    x[e] = v;
  }
}

int main(int argc, char** argv) {
  const char* names[] = {"potrf", "trsm", "syrk", "gemm", "geqrt", "larfb", "tsqrt", "ssrfb", "getrf", "gessm", "tstrf", "ssssm"};
  if (argc < 4) { fprintf(stderr, "usage: kbench kind b ib [ctas reps]\n"); return 1; }
  int kind = -1;
  for (int i = 0; i < 12; ++i) if (!strcmp(argv[1], names[i])) kind = i;
  const int b = atoi(argv[2]), ib = atoi(argv[3]);
  const int cps = argc > 4 ? atoi(argv[4]) : 1;
  const int reps = argc > 5 ? atoi(argv[5]) : 4;
  const int shared_ab = argc > 6 ? atoi(argv[6]) : 0;
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int grid = kind == 0 || kind == 4 || kind == 6 || kind == 8 || kind == 10 ? sms * cps : sms * cps;
  const size_t bb = (size_t)b * b;
  double *tiles, *aux, *scratch; int* ipiv;
  const size_t scr = ((size_t)2 * ib * b + 64 + 31) & ~(size_t)31;
  CK(cudaMalloc(&tiles, grid * 3 * bb * sizeof(double)));
  CK(cudaMalloc(&aux, grid * (size_t)ib * b * sizeof(double)));
  CK(cudaMalloc(&scratch, grid * scr * sizeof(double)));
  CK(cudaMalloc(&ipiv, grid * (size_t)b * sizeof(int)));
  CK(cudaMemset(aux, 0, grid * (size_t)ib * b * sizeof(double)));
  // identity-ish pivots (no swaps) for gessm / ssssm
  std::vector<int> hp(grid * (size_t)b);
  for (size_t x = 0; x < hp.size(); ++x) hp[x] = (int)(x % b) + 1;
  CK(cudaMemcpy(ipiv, hp.data(), hp.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(kb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_DOUBLES * 8));
  init_kernel<<<1024, 256>>>(tiles, grid * 3 * bb, b, kind);
  CK(cudaDeviceSynchronize());
  kb_kernel<<<grid, TF_THREADS, SMEM_DOUBLES * 8>>>(kind, b, ib, tiles, aux, ipiv, scratch, scr, 1, shared_ab);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kb_kernel<<<grid, TF_THREADS, SMEM_DOUBLES * 8>>>(kind, b, ib, tiles, aux, ipiv, scratch, scr, reps, shared_ab);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
#ifdef TF_PROBE
  {
    unsigned long long* pr;
    cudaMallocManaged(&pr, 8 * sizeof(unsigned long long));
    for (int i = 0; i < 8; ++i) pr[i] = 0;
    cudaMemcpyToSymbol(g_probe, &pr, sizeof(pr));
    kb_kernel<<<grid, TF_THREADS, SMEM_DOUBLES * 8>>>(kind, b, ib, tiles, aux, ipiv, scratch, scr, reps, shared_ab);
    CK(cudaDeviceSynchronize());
    printf("probe us/item:");
    for (int i = 0; i < 8; ++i) printf(" [%d] %.2f", i, pr[i] / 1e3 / grid / reps);
    printf("\n");
  }
#endif
#ifdef TF_PROF_LU
  {
    long long z[32] = {0}, h[32];
    cudaMemcpyToSymbol(g_lu_prof, z, sizeof(z));
    kb_kernel<<<grid, TF_THREADS, SMEM_DOUBLES * 8>>>(kind, b, ib, tiles, aux, ipiv, scratch, scr, reps, shared_ab);
    CK(cudaDeviceSynchronize());
    cudaMemcpyFromSymbol(h, g_lu_prof, sizeof(h));
    printf("lu phases us/task:");
    for (int i = 0; i < 32; ++i) if (h[i]) printf(" [%d] %.1f", i, h[i] / 1.92e3 / grid / reps);
    printf("\n");
  }
#endif
  const double fl_task[] = {b * (double)b * b / 3, (double)b * b * b, (double)b * b * (b + 1.0), 2.0 * b * b * b,
                            4.0 * b * b * b / 3, 2.0 * b * b * b + 3.0 * ib * b * b, 2.0 * b * b * b + (double)ib * b * b,
                            4.0 * b * b * b + (double)ib * b * b, 2.0 * b * b * b / 3, (double)b * b * b,
                            (double)b * b * b + ib * (double)b * b / 2, 2.0 * b * b * b + (double)ib * b * b};
  const double fl = fl_task[kind] / items_of(kind, b, ib) * (double)grid * reps;
  const double us_item = ms * 1e3 / reps;
  printf("{\"kind\": \"%s\", \"b\": %d, \"ib\": %d, \"grid\": %d, \"reps\": %d, \"ms\": %.3f, \"us_per_item\": %.2f, "
         "\"gflops_per_sm\": %.2f, \"tflops\": %.3f}\n",
         names[kind], b, ib, grid, reps, ms, us_item, fl / (ms * 1e-3) / 1e9 / (grid / cps) , fl / (ms * 1e-3) / 1e12);
  return 0;
}
