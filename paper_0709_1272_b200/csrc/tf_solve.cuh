// tf_solve.cuh — tile kernels of the solve / apply routines: solving
// with the tiled factors and applying N for the GETWP stability study.
//
// The forward halves of the solves reuse the factorization's own update kernels on the
// right-hand-side tiles X(k,c) as if they were extra tile columns of the matrix: DGESSM /
// DSSSSM apply N^{-1} (Algorithm 3 on columns right of panel k), DLARFB / DSSRFB apply Q^T
// (Algorithm 2).  The kernels here are the remaining pieces:
//   unitl_item    explicit unit-lower copy of a factored diagonal tile (the operand DGESSM /
//                 DLARFB read; during a factorization the panel kernels write it)
//   trsmu_item    X(k,c) <- U_kk^{-1} X(k,c), U upper non-unit (back substitution, blocked
//                 by 32 rows from the bottom; rows above updated on the DMMA engine)
//   xgemm_item    X(i,c) -= U_ik X(k,c) (DMMA engine)
//   unssssm_item  inverse of one DSSSSM step (C4: x2 += L_ik[:,s] x1, x1 <- (I + Ls_s) x1,
//                 then the block's swaps undone in reverse order), blocks s = t-1..0
//   ungessm_item  inverse of DGESSM (x <- L_kk x, then the interchanges undone in reverse)
// Work items are 32-column slabs of an X tile (64 for xgemm).  These kernels serve the
// solves and the stability lab, not the factorization hot path: they are written for
// clarity and any b (incl. b = n = 2048 of the lab's p = 1 case).
#pragma once

namespace tf {

__device__ inline void unitl_item(const Ctx& cx, const double* A, double* VX) {
  const int b = cx.b;
  const size_t bb = (size_t)b * b;
  for (size_t e = threadIdx.x; e < bb; e += TF_THREADS) {
    const int r = (int)(e % b), c = (int)(e / b);
    VX[e] = (r > c) ? ldg_cg(A + e) : (r == c ? 1.0 : 0.0);
  }
}

// X(:, slab) <- U^{-1} X(:, slab); U: upper triangle of the b x b tile (column-major).
__device__ inline void trsmu_item(const Ctx& cx, const double* U, double* X, int item, double* sm) {
  const int b = cx.b, tid = threadIdx.x;
  const int c0 = item * 32, nc = min(32, b - c0);
  X += (size_t)c0 * b;
  double* sUb = sm;             // 32 x 33: U block, (r, m) at r*33 + m
  double* sX = sUb + 32 * 33;   // 32 x 33: X block rows, (r, c) at r*33 + c
  for (int r1 = b; r1 > 0;) {
    const int nb = (r1 % 32) ? r1 % 32 : 32, r0 = r1 - nb;
    for (int e = tid; e < 32 * 32; e += TF_THREADS) {
      const int r = e % 32, m = e / 32;
      sUb[r * 33 + m] = (r < nb && m < nb && r <= m) ? ldg_cg(U + (r0 + r) + (size_t)(r0 + m) * b) : 0.0;
      sX[r * 33 + m] = (r < nb && m < nc) ? ldg_cg(X + (r0 + r) + (size_t)m * b) : 0.0;
    }
    __syncthreads();
    {
      const int c = tid >> 4, l = tid & 15;  // 16 lanes per column
      for (int r = nb - 1; r >= 0; --r) {
        __syncwarp();
        const double xr = sX[r * 33 + c] / sUb[r * 33 + r];
        __syncwarp();
        if (l == 0) sX[r * 33 + c] = xr;
        for (int m = l; m < r; m += 16) sX[m * 33 + c] -= sUb[m * 33 + r] * xr;
      }
    }
    __syncthreads();
    for (int e = tid; e < nb * nc; e += TF_THREADS) {
      const int r = e % nb, c = e / nb;
      X[(r0 + r) + (size_t)c * b] = sX[r * 33 + c];
    }
    __syncthreads();
    if (r0 > 0) {
      // rows above the block: X[0:r0, slab] -= U[0:r0, r0:r1] X[r0:r1, slab]
      update_mn(sm, X, b, U + (size_t)r0 * b, b, X + r0, b, r0, nc, nb);
      __syncthreads();
    }
    r1 = r0;
  }
}

// C(:, slab) -= A B(:, slab), all b x b column-major tiles; slabs of 64 columns.
__device__ inline void xgemm_item(const Ctx& cx, const double* A, const double* B, double* C, int item, double* sm) {
  const int b = cx.b;
  const int n0 = item * 64, nc = min(64, b - n0);
  update_mn(sm, C + (size_t)n0 * b, b, A, b, B + (size_t)n0 * b, b, b, nc, b);
  __syncthreads();
}

// Inverse of DSSSSM on a 32-column slab of [X1; X2] (C4 of SURVEY §8(c), the oracle's
// o_lu_apply_N step): blocks s = t-1..0: x2 += L[:, s] x1_s; x1_s <- (I + Ls_s) x1_s (both
// from the block's original x1_s); then the block's pairwise swaps undone, j descending.
__device__ inline void unssssm_item(const Ctx& cx, const double* L, const double* Ls, const int* ipiv, double* X1,
                                    double* X2, int item, double* sm) {
  const int b = cx.b, ib = cx.ib, tid = threadIdx.x;
  const int c0 = item * 32, nc = min(32, b - c0);
  X1 += (size_t)c0 * b;
  X2 += (size_t)c0 * b;
  double* sX1 = sm;  // ib x 33
  for (int s = b / ib - 1; s >= 0; --s) {
    const int cb0 = s * ib;
    for (int e = tid; e < ib * 32; e += TF_THREADS) {
      const int m = e % ib, c = e / ib;
      sX1[m * 33 + c] = c < nc ? ldg_cg(X1 + (cb0 + m) + (size_t)c * b) : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < b * nc; e += TF_THREADS) {
      const int r = e % b, c = e / b;
      double acc = 0.0;
      for (int m = 0; m < ib; ++m) acc += ldg_cg(L + r + (size_t)(cb0 + m) * b) * sX1[m * 33 + c];
      X2[r + (size_t)c * b] = ldg_cg(X2 + r + (size_t)c * b) + acc;
    }
    for (int e = tid; e < ib * nc; e += TF_THREADS) {
      const int r = e % ib, c = e / ib;
      double acc = 0.0;
      for (int m = 0; m < r; ++m) acc += ldg_cg(Ls + r + (size_t)(cb0 + m) * ib) * sX1[m * 33 + c];
      X1[(cb0 + r) + (size_t)c * b] = sX1[r * 33 + c] + acc;
    }
    __syncthreads();
    if (tid < nc)
      for (int j = cb0 + ib - 1; j >= cb0; --j) {
        const int pv = ipiv[j];
        if (pv > b) {
          double* p1 = X1 + j + (size_t)tid * b;
          double* p2 = X2 + (pv - b - 1) + (size_t)tid * b;
          const double t = *p1;
          *p1 = *p2;
          *p2 = t;
        }
      }
    __syncthreads();
  }
}

// Inverse of DGESSM on a 32-column slab: x <- L_kk x (unit lower; rows from the bottom so
// every row's dot uses the original rows above it), then the interchanges j = b-1..0 undone.
__device__ inline void ungessm_item(const Ctx& cx, const double* F, const int* ipiv, double* X, int item,
                                    double* sm) {
  const int b = cx.b, tid = threadIdx.x;
  const int c0 = item * 32, nc = min(32, b - c0);
  X += (size_t)c0 * b;
  const int c = tid >> 4, l = tid & 15;  // 16 lanes per column
  for (int r = b - 1; r >= 1; --r) {
    double acc = 0.0;
    if (c < nc)
      for (int m = l; m < r; m += 16) acc += ldg_cg(F + r + (size_t)m * b) * ldg_cg(X + m + (size_t)c * b);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (c < nc && l == 0) X[r + (size_t)c * b] = ldg_cg(X + r + (size_t)c * b) + acc;
    __syncthreads();
  }
  if (tid < nc)
    for (int j = b - 1; j >= 0; --j) {
      const int r = ipiv[j] - 1;
      if (r != j) {
        double* p1 = X + j + (size_t)tid * b;
        double* p2 = X + r + (size_t)tid * b;
        const double t = *p1;
        *p1 = *p2;
        *p2 = t;
      }
    }
  __syncthreads();
}

}  // namespace tf
