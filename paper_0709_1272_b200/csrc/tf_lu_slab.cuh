// tf_lu_slab.cuh — register-resident slab kernels for the LU update tasks on sm_100a
// (b in {128, 256, 512}, ib in {32, 64}; same slab layout as tf_qr_slab.cuh: a work item
// owns 32 columns of a tile in FP64 DMMA accumulators, warp w holding rows
// [w*b/16, (w+1)*b/16)).
//
//   ssssm_reg  SSSSM: for each inner block s of the pairwise-pivoted
//              panel, [U_s; A] <- swaps (top row jj <-> bottom row r, in pivot order),
//              U_s <- (I + Ls_s)^{-1} U_s (unit-lower forward substitution, subtraction order
//              m = 0..r-1 as in the oracle), A -= L_ik[:, s] U_s on the tensor pipe.  Only the
//              A rows that a pivot names leave the registers (through shared memory).
//   gessm_reg  GESSM: A_kj <- L_kk^{-1} P_kk A_kj — the row permutation
//              composed from the b interchanges is applied through shared memory once, then
//              per block: forward substitution of the block rows, and the rows below are
//              updated by DMMA from the resident registers.
#pragma once
#include "tf_qr_slab.cuh"

namespace tf {

constexpr int LU_LDW = NSR + 4;  // row stride of U_s / gathered rows in smem (conflict-free B fragments)

// Forward substitution U_s <- (I + L)^{-1} U_s for ib rows x NSR columns held in smem
// (sU[m*LU_LDW + c]); sL[r*(ib+1) + m] = L(r, m), r > m.  16 lanes per column (two columns
// per warp), right-looking over m.
__device__ __forceinline__ void lu_block_solve(double* sU, const double* sL, int ib) {
  const int c = threadIdx.x >> 4, l = threadIdx.x & 15;
  for (int m = 0; m < ib; ++m) {
    __syncwarp();
    const double xm = sU[m * LU_LDW + c];
    for (int r = m + 1 + l; r < ib; r += 16) sU[r * LU_LDW + c] -= sL[r * (ib + 1) + m] * xm;
  }
  __syncwarp();
}

// SSSSM item: 32 columns of [U_kj; A_ij].  L = A_ik (multipliers), Ls = L strip (i,k),
// ipiv = pivots (i,k) in [1, 2b] (b + r + 1 = bottom row r swapped in).
template <int MI>
__device__ inline void ssssm_reg(const Ctx& cx, const double* L, const double* Ls, const int* ipiv, double* U,
                                 double* A, int item, double* sm) {
  constexpr int RW = 8 * MI;
  const int b = cx.b, ib = cx.ib;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  const int r0 = warp * RW;
  U += (size_t)item * NSR * b;
  A += (size_t)item * NSR * b;
  double* sU = sm;                              // ib x LU_LDW: U_s
  double* sA = sU + 64 * LU_LDW;                // ib slots x LU_LDW: the A rows the pivots name
  double* sL = sA + 64 * LU_LDW;                // ib x (ib+1): L(r, m), r > m
  int* flag = reinterpret_cast<int*>(sL + 64 * 65);  // b: slot of bottom row r (INT_MAX = none)
  int* spv = flag + 512;                        // ib pivots of the block
  double acc[MI][SNJ][2];
  slab_load<MI>(acc, A, b);
  for (int c0 = 0; c0 < b; c0 += ib) {
    for (int r = tid; r < b; r += TF_THREADS) flag[r] = INT_MAX;
    for (int e = tid; e < ib * NSR; e += TF_THREADS) {
      const int m = e % ib, c = e / ib;
      sU[m * LU_LDW + c] = ldg_cg(U + (c0 + m) + (size_t)c * b);
    }
    for (int e = tid; e < ib * ib; e += TF_THREADS) {
      const int r = e % ib, m = e / ib;
      sL[r * (ib + 1) + m] = (r > m) ? ldg_cg(Ls + (size_t)c0 * ib + e) : 0.0;
    }
    __syncthreads();
    if (tid < ib) {
      const int pv = ipiv[c0 + tid];
      spv[tid] = pv;
      if (pv > b) atomicMin(&flag[pv - b - 1], tid);  // slot = first pivot naming the row
    }
    __syncthreads();
    // named A rows: registers -> smem slots
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int f = flag[r0 + 8 * i + g];
      if (f != INT_MAX)
#pragma unroll
        for (int j = 0; j < SNJ; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) sA[f * LU_LDW + 8 * j + 2 * q + e] = acc[i][j][e];
    }
    __syncthreads();
    // pairwise swaps in pivot order, then the unit-lower solve (per column)
    {
      const int c = tid >> 4;
      if ((tid & 15) == 0)
        for (int jj = 0; jj < ib; ++jj) {
          const int pv = spv[jj];
          if (pv > b) {
            const int f = flag[pv - b - 1];
            const double t = sU[jj * LU_LDW + c];
            sU[jj * LU_LDW + c] = sA[f * LU_LDW + c];
            sA[f * LU_LDW + c] = t;
          }
        }
      lu_block_solve(sU, sL, ib);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int f = flag[r0 + 8 * i + g];
      if (f != INT_MAX)
#pragma unroll
        for (int j = 0; j < SNJ; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) acc[i][j][e] = sA[f * LU_LDW + 8 * j + 2 * q + e];
    }
    for (int e = tid; e < ib * NSR; e += TF_THREADS) {
      const int m = e % ib, c = e / ib;
      U[(c0 + m) + (size_t)c * b] = sU[m * LU_LDW + c];
    }
    // A -= L[:, c0:c0+ib] U_s
    for (int ks = 0; ks < ib / 4; ++ks) {
      double a[MI], bq[SNJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = -L[(r0 + 8 * i + g) + (size_t)(c0 + 4 * ks + q) * b];
#pragma unroll
      for (int j = 0; j < SNJ; ++j) bq[j] = sU[(4 * ks + q) * LU_LDW + 8 * j + g];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < SNJ; ++j) dmma(acc[i][j], a[i], bq[j]);
    }
    __syncthreads();
  }
  slab_store<MI>(acc, A, b);
}

// GESSM item: 32 columns of C = A_kj <- L_kk^{-1} P_kk C.  LX = explicit unit-lower L_kk
// copy (b x b), ipiv = GETRF interchanges in [1, b] (LAPACK form, Z12).
template <int MI>
__device__ inline void gessm_reg(const Ctx& cx, const double* LX, const int* ipiv, double* C, int item,
                                 double* sm) {
  constexpr int RW = 8 * MI;
  const int b = cx.b, ib = cx.ib;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  const int r0 = warp * RW;
  C += (size_t)item * NSR * b;
  double* sC = sm;                              // b x LU_LDW (permutation staging)
  double* sU = sm;                              // ib x LU_LDW (after the permutation)
  double* sL = sU + 64 * LU_LDW;                // ib x (ib+1)
  int* perm = reinterpret_cast<int*>(sm + 512 * LU_LDW);
  double acc[MI][SNJ][2];
  slab_load<MI>(acc, C, b);
  // P_kk: compose the b sequential interchanges into a gather permutation
  for (int r = tid; r < b; r += TF_THREADS) perm[r] = r;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < SNJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) sC[(r0 + 8 * i + g) * LU_LDW + 8 * j + 2 * q + e] = acc[i][j][e];
  __syncthreads();
  if (tid == 0)
    for (int j = 0; j < b; ++j) {
      const int r = ipiv[j] - 1;
      const int t = perm[j];
      perm[j] = perm[r];
      perm[r] = t;
    }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int src = perm[r0 + 8 * i + g];
#pragma unroll
    for (int j = 0; j < SNJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) acc[i][j][e] = sC[src * LU_LDW + 8 * j + 2 * q + e];
  }
  __syncthreads();
  // blocked unit-lower forward solve
  for (int c0 = 0; c0 < b; c0 += ib) {
    const int c1 = c0 + ib;
    // block rows -> smem (their owner warps), L block
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int row = r0 + 8 * i + g;
      if (row >= c0 && row < c1)
#pragma unroll
        for (int j = 0; j < SNJ; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) sU[(row - c0) * LU_LDW + 8 * j + 2 * q + e] = acc[i][j][e];
    }
    for (int e = tid; e < ib * ib; e += TF_THREADS) {
      const int r = e % ib, m = e / ib;
      sL[r * (ib + 1) + m] = (r > m) ? ldg_cg(LX + (c0 + r) + (size_t)(c0 + m) * b) : 0.0;
    }
    __syncthreads();
    lu_block_solve(sU, sL, ib);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int row = r0 + 8 * i + g;
      if (row >= c0 && row < c1)
#pragma unroll
        for (int j = 0; j < SNJ; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) acc[i][j][e] = sU[(row - c0) * LU_LDW + 8 * j + 2 * q + e];
    }
    // rows below the block: C -= L[:, c0:c1] C_s
    if (c1 < b && r0 + RW > c1) {
      for (int ks = 0; ks < ib / 4; ++ks) {
        double a[MI], bq[SNJ];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int row = r0 + 8 * i + g;
          a[i] = row >= c1 ? -LX[row + (size_t)(c0 + 4 * ks + q) * b] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < SNJ; ++j) bq[j] = sU[(4 * ks + q) * LU_LDW + 8 * j + g];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < SNJ; ++j) dmma(acc[i][j], a[i], bq[j]);
      }
    }
    __syncthreads();
  }
  slab_store<MI>(acc, C, b);
}

}  // namespace tf
