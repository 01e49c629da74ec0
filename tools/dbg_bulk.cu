// dbg_bulk.cu — single-CTA harness for the mbarrier/bulk-copy GEMM pipeline.
// Runs consecutive Gemm::run calls with varying K (as TRSM/POTRF do) and checks results.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_0709_1272_b200/csrc/tf_kernels.cuh"
using namespace tf;

template <class G>
__global__ void __launch_bounds__(TF_THREADS, 1) dbg_kernel(const double* A, const double* B, double* C, int ld,
                                                            int kmax, int step, int* progress, int mode) {
  extern __shared__ __align__(16) double sm[];
  pipe_init(sm);
  for (int K = step; K <= kmax; K += step) {
    if (mode & 1) {  // generic stores into the A operand columns the next call reads
      double* Aw = const_cast<double*>(A);
      for (int e = threadIdx.x; e < 128 * step; e += TF_THREADS) Aw[(e % 128) + (size_t)(K - step + e / 128) * ld] += 0.0;
      __syncthreads();
    }
    if (mode & 2) {  // shared-memory writes beyond the pipeline's buffers
      for (int e = threadIdx.x; e < 1024; e += TF_THREADS) sm[G::SMEM_DOUBLES + e] = 1.0;
      __syncthreads();
    }
    G g;
    g.zero();
    if (threadIdx.x == 0) { atomicExch(progress, K); __threadfence_system(); }
    g.run(sm, A, ld, (mode & 4) ? B + K : B, ld, 128, G::BN_, K);
    g.for_each(128, 1 << 20, [&](int r, int c, double v) { C[r + (size_t)c * ld + (size_t)(K / step - 1) * ld * ld] = v; });
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicExch(progress, -1);
}

__device__ void trsm_copy(int b, const double* L, double* X, double* sm, int mode) {
  double* D = sm + GemmNT32::SMEM_DOUBLES;
  for (int jb = 0; jb < b; jb += NB) {
    const int nb = min(NB, b - jb);
    if (jb > 0) {
      GemmNT32 g;
      g.zero();
      g.run(sm, X, b, L + jb, b, 128, nb, jb);
      if (!(mode & 1)) sub_store(g, X + (size_t)jb * b, b, 128, nb);
    }
    if (!(mode & 2)) load_lower_block(D, L + jb + (size_t)jb * b, b, nb);
    if (!(mode & 4)) row_solve(X + (size_t)jb * b, b, 128, nb, D);
    __syncthreads();
    if (threadIdx.x == 0) printf("jb %d done\n", jb);
  }
}
__global__ void __launch_bounds__(TF_THREADS, 1) dbg_trsm2(const double* L, double* X, int b, int mode) {
  extern __shared__ __align__(16) double sm[];
  pipe_init(sm);
  trsm_copy(b, L, X, sm, mode);
}

__global__ void __launch_bounds__(TF_THREADS, 1) dbg_trsm(const double* L, double* X, int b, int item, int* progress) {
  extern __shared__ __align__(16) double sm[];
  Ctx cx; cx.b = b; cx.ib = 32; cx.scratch = nullptr; cx.info = nullptr; cx.abort_flag = nullptr;
  pipe_init(sm);
  if (item >= 0) trsm_item(cx, L, X, item, sm);
  else potrf_item(cx, X, sm);
  if (threadIdx.x == 0) atomicExch(progress, -1);
}

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 't') {
    const int b = atoi(argv[2]), item = atoi(argv[3]);
    double *L, *X; int* prog;
    cudaMalloc(&L, b * b * 8); cudaMalloc(&X, b * b * 8); cudaMallocManaged(&prog, 4); *prog = 0;
    std::vector<double> h(b * b);
    for (int i = 0; i < b * b; ++i) h[i] = ((i % b) == (i / b)) ? 4.0 + b : 0.01 * ((i % 11) - 5);
    cudaMemcpy(L, h.data(), b * b * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(X, h.data(), b * b * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(dbg_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_DOUBLES * 8);
    if (argc > 4) {
      cudaFuncSetAttribute(dbg_trsm2, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_DOUBLES * 8);
      dbg_trsm2<<<1, TF_THREADS, SMEM_DOUBLES * 8>>>(L, X, b, atoi(argv[4]));
    } else
    dbg_trsm<<<1, TF_THREADS, SMEM_DOUBLES * 8>>>(L, X, b, item, prog);
    for (int t = 0; t < 400; ++t) {
      if (cudaStreamQuery(0) == cudaSuccess) break;
      struct timespec ts = {0, 50 * 1000 * 1000};
      nanosleep(&ts, nullptr);
    }
    printf("query: %s\n", cudaGetErrorString(cudaStreamQuery(0)));
    printf("progress=%d\n", *(volatile int*)prog);
    return 0;
  }
  const int which = argc > 1 ? atoi(argv[1]) : 32;
  const int ld = argc > 5 ? atoi(argv[5]) : 512, kmax = argc > 2 ? atoi(argv[2]) : 128, step = argc > 3 ? atoi(argv[3]) : 32;
  double *A, *B, *C;
  int* prog;
  cudaMalloc(&A, ld * ld * 8);
  cudaMalloc(&B, ld * ld * 8);
  const int ncalls = kmax / step;
  cudaMalloc(&C, (size_t)ncalls * ld * ld * 8);
  cudaMallocManaged(&prog, 4);
  std::vector<double> hA(ld * ld), hB(ld * ld);
  for (int i = 0; i < ld * ld; ++i) { hA[i] = (i % 7) - 3; hB[i] = (i % 5) - 2; }
  cudaMemcpy(A, hA.data(), ld * ld * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB.data(), ld * ld * 8, cudaMemcpyHostToDevice);
  *prog = 0;
  int N;
  if (which == 32) {
    cudaFuncSetAttribute(dbg_kernel<GemmNT32>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_DOUBLES * 8);
    dbg_kernel<GemmNT32><<<1, TF_THREADS, SMEM_DOUBLES * 8>>>(A, B, C, ld, kmax, step, prog, argc > 4 ? atoi(argv[4]) : 0);
    N = 32;
  } else {
    cudaFuncSetAttribute(dbg_kernel<GemmNT128>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_DOUBLES * 8);
    dbg_kernel<GemmNT128><<<1, TF_THREADS, SMEM_DOUBLES * 8>>>(A, B, C, ld, kmax, step, prog, argc > 4 ? atoi(argv[4]) : 0);
    N = 128;
  }
  for (int t = 0; t < 100; ++t) {
    if (cudaStreamQuery(0) == cudaSuccess) break;
    struct timespec ts = {0, 50 * 1000 * 1000};
    nanosleep(&ts, nullptr);
    printf("poll %d progress K=%d\n", t, *(volatile int*)prog);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("done: %s progress=%d\n", cudaGetErrorString(e), *prog);
  std::vector<double> hC((size_t)ncalls * ld * ld);
  cudaMemcpy(hC.data(), C, hC.size() * 8, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int call = 0; call < ncalls; ++call) {
    const int K = step * (call + 1);
    for (int c = 0; c < N; ++c)
      for (int r = 0; r < 128; ++r) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += hA[r + k * ld] * hB[c + k * ld];
        double g = hC[(size_t)call * ld * ld + r + (size_t)c * ld];
        if (fabs(g - s) > maxerr) maxerr = fabs(g - s);
      }
  }
  printf("maxerr %g\n", maxerr);
  return 0;
}
