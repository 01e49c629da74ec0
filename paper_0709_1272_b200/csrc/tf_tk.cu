// tf_tk.cu — the per-kernel test launcher (tk_run in the C-ABI): one CTA per work item of
// a single tile task, running the same device functions as the persistent scheduler
// (tf_device.cu).  A separate translation unit so the two big kernels compile in parallel.
#include <cuda_runtime.h>

#include "tf_kernels.cuh"
#include "tf_sched.h"

namespace tf {

// Per-kernel test launcher: one CTA per work item of a single task.
__global__ void __launch_bounds__(TF_THREADS, 1)
    tk_kernel(int kind, int b, int ib, double* t0, double* t1, double* t2, double* aux, int* ipiv, double* vx,
              double* scratch, size_t scr_stride, int* info) {
  extern __shared__ __align__(16) double sm[];
  Ctx cx;
  cx.b = b;
  cx.ib = ib;
  cx.scratch = scratch + (size_t)blockIdx.x * scr_stride;
  cx.info = info;
  cx.abort_flag = nullptr;
  cx.nopiv = 0;
  pipe_init(sm);
  const int sub = blockIdx.x;
  int f = -1;
  switch (kind) {
    case 0: f = potrf_item(cx, t0, sm); break;
    case 1: trsm_item(cx, t0, t1, sub, sm); break;
    case 2: syrk_item(cx, t0, t1, sub, sm); break;
    case 3: gemm_item(cx, t0, t1, t2, sub, sm); break;
    case 4: geqrt_item(cx, t0, aux, vx, sm); break;
    case 5: larfb_item(cx, vx, aux, t1, sub, sm); break;
    case 6: tsqrt_item(cx, t0, t1, aux, sm); break;
    case 7: ssrfb_item(cx, t0, aux, t1, t2, sub, sm); break;
    case 8: f = getrf_item(cx, t0, ipiv, vx, sm); break;
    case 9: gessm_item(cx, vx, ipiv, t1, sub, sm); break;
    case 10: f = tstrf_item(cx, t0, t1, aux, ipiv, sm); break;
    case 11: ssssm_item(cx, t0, aux, ipiv, t1, t2, sub, sm); break;
  }
  if (info && threadIdx.x == 0 && blockIdx.x == 0) *info = (f >= 0) ? f + 1 : 0;
}

// unit-lower explicit copy (V_kk / L_kk) of a factored diagonal tile, for tk_run
__global__ void unit_lower_kernel(const double* A, double* X, int b) {
  const size_t bb = (size_t)b * b;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < bb; e += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % b), c = (int)(e / b);
    X[e] = (r > c) ? A[e] : (r == c ? 1.0 : 0.0);
  }
}


static int ok_or_tk(cudaError_t e) { return e == cudaSuccess ? 0 : (int)e; }

int tk_kernel_setup(size_t smem) {
  return ok_or_tk(cudaFuncSetAttribute(tk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}
int launch_tk(int kind, int b, int ib, double* t0, double* t1, double* t2, double* aux, int* ipiv, double* vx,
              double* scratch, size_t scr_stride, int* info, int items, size_t smem, void* stream) {
  tk_kernel<<<items, TF_THREADS, smem, (cudaStream_t)stream>>>(kind, b, ib, t0, t1, t2, aux, ipiv, vx, scratch,
                                                               scr_stride, info);
  return ok_or_tk(cudaGetLastError());
}
int launch_unit_lower(const double* A, double* X, int b, void* stream) {
  unit_lower_kernel<<<64, 256, 0, (cudaStream_t)stream>>>(A, X, b);
  return ok_or_tk(cudaGetLastError());
}

}  // namespace tf
