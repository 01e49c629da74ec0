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
template <int R>
__device__ __forceinline__ void lu_block_solve_reg(double* sU, const double* sL) {
  // rows l + 16 t (t < R) in registers; row m broadcast by shuffle within the 16-lane group
  // (the same operations in the same order as the shared-memory loop)
  constexpr int IB = 16 * R;
  const int c = threadIdx.x >> 4, l = threadIdx.x & 15;
  const int base = threadIdx.x & 16;
  double x[R];
#pragma unroll
  for (int t = 0; t < R; ++t) x[t] = sU[(l + 16 * t) * LU_LDW + c];
#pragma unroll
  for (int m = 0; m < IB; ++m) {
    const double xm = __shfl_sync(0xffffffffu, x[m >> 4], base | (m & 15));
#pragma unroll
    for (int t = m >> 4; t < R; ++t)
      if (l + 16 * t > m) x[t] -= sL[(l + 16 * t) * (IB + 1) + m] * xm;
  }
#pragma unroll
  for (int t = 0; t < R; ++t) sU[(l + 16 * t) * LU_LDW + c] = x[t];
  __syncwarp();
}

__device__ __forceinline__ void lu_block_solve(double* sU, const double* sL, int ib) {
  if (ib == 32) { lu_block_solve_reg<2>(sU, sL); return; }
  if (ib == 64) { lu_block_solve_reg<4>(sU, sL); return; }
  const int c = threadIdx.x >> 4, l = threadIdx.x & 15;
  for (int m = 0; m < ib; ++m) {
    __syncwarp();
    const double xm = sU[m * LU_LDW + c];
    for (int r = m + 1 + l; r < ib; r += 16) sU[r * LU_LDW + c] -= sL[r * (ib + 1) + m] * xm;
  }
  __syncwarp();
}

#ifdef TF_PROF_LU
__device__ long long g_lu_prof[16];
#define TF_LU_T0() long long lu_t_ = clock64()
#define TF_LU_T(k)                                                       \
  do {                                                                   \
    if (threadIdx.x == 0) {                                              \
      const long long t_ = clock64();                                    \
      atomicAdd(reinterpret_cast<unsigned long long*>(&g_lu_prof[k]), (unsigned long long)(t_ - lu_t_)); \
      lu_t_ = t_;                                                        \
    }                                                                    \
  } while (0)
#else
#define TF_LU_T0() (void)0
#define TF_LU_T(k) (void)0
#endif

// One inner block of the pairwise-pivoted update on a register slab (SSSSM step):
// [U_s; A] <- swaps of block s, U_s <- (I + Ls_s)^{-1} U_s, A -= L[:, s] U_s.
//   Us  : U rows c0.. of the slab columns, (m, c) at Us[m + c*b] (read, then written back)
//   Lc  : L columns of the block, (r, m) at Lc[r + m*b]
//   Lsb : Ls block s, (r, m) at Lsb[r + m*ib];  pv: the block's ib pivots (1-based, [1, 2b])
template <int MI>
__device__ __forceinline__ void lu_ts_apply(double (&acc)[MI][SNJ][2], double* Us, const double* Lc, const double* Lsb,
                                            const int* pv, int ib, int b, double* sm) {
  constexpr int RW = 8 * MI;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  const int r0 = warp * RW;
  double* sU = sm;                              // ib x LU_LDW: U_s
  double* sA = sU + 64 * LU_LDW;                // ib slots x LU_LDW: the A rows the pivots name
  double* sL = sA + 64 * LU_LDW;                // ib x (ib+1): L(r, m), r > m
  int* flag = reinterpret_cast<int*>(sL + 64 * 65);  // b: slot of bottom row r (INT_MAX = none)
  int* spv = flag + 512;                        // ib pivots of the block
  for (int r = tid; r < b; r += TF_THREADS) flag[r] = INT_MAX;
  for (int e = tid; e < ib * NSR; e += TF_THREADS) {
    const int m = e % ib, c = e / ib;
    sU[m * LU_LDW + c] = ldg_cg(Us + m + (size_t)c * b);
  }
  for (int e = tid; e < ib * ib; e += TF_THREADS) {
    const int r = e % ib, m = e / ib;
    sL[r * (ib + 1) + m] = (r > m) ? ldg_cg(Lsb + e) : 0.0;
  }
  __syncthreads();
  if (tid < ib) {
    const int v = pv[tid];
    spv[tid] = v;
    if (v > b) atomicMin(&flag[v - b - 1], tid);  // slot = first pivot naming the row
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
        const int v = spv[jj];
        if (v > b) {
          const int f = flag[v - b - 1];
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
    Us[m + (size_t)c * b] = sU[m * LU_LDW + c];
  }
  // A -= L[:, block] U_s
  for (int ks = 0; ks < ib / 4; ++ks) {
    double a[MI], bq[SNJ];
#pragma unroll
    for (int i = 0; i < MI; ++i) a[i] = -Lc[(r0 + 8 * i + g) + (size_t)(4 * ks + q) * b];
#pragma unroll
    for (int j = 0; j < SNJ; ++j) bq[j] = sU[(4 * ks + q) * LU_LDW + 8 * j + g];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < SNJ; ++j) dmma(acc[i][j], a[i], bq[j]);
  }
  __syncthreads();
}

// SSSSM item: 32 columns of [U_kj; A_ij].  L = A_ik (multipliers), Ls = L strip (i,k),
// ipiv = pivots (i,k) in [1, 2b] (b + r + 1 = bottom row r swapped in).
template <int MI>
__device__ inline void ssssm_reg(const Ctx& cx, const double* L, const double* Ls, const int* ipiv, double* U,
                                 double* A, int item, double* sm) {
  const int b = cx.b, ib = cx.ib;
  U += (size_t)item * NSR * b;
  A += (size_t)item * NSR * b;
  double acc[MI][SNJ][2];
  slab_load<MI>(acc, A, b);
  for (int c0 = 0; c0 < b; c0 += ib)
    lu_ts_apply<MI>(acc, U + c0, L + (size_t)c0 * b, Ls + (size_t)c0 * ib, ipiv + c0, ib, b, sm);
  slab_store<MI>(acc, A, b);
}

// Row interchanges j <-> ipiv[j]-1, j = j0..j1-1 in order (LAPACK form), applied to the
// register slab: composed into a gather permutation, applied through shared memory.
template <int MI>
__device__ __forceinline__ void lu_rows_permute(double (&acc)[MI][SNJ][2], const int* ipiv, int j0, int j1, int b,
                                                double* sm, int tp = -1) {
  constexpr int RW = 8 * MI;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  const int r0 = warp * RW;
  double* sC = sm;                                        // b x LU_LDW
  int* perm = reinterpret_cast<int*>(sm + 512 * LU_LDW);  // b
  int* spv = perm + 512;                                  // the interchanges, staged
  if (tp >= 0) {
    if (tid < b) perm[tid] = tp;  // (the caller's running composition, row tid <- row tp)
  } else {
    for (int r = tid; r < b; r += TF_THREADS) perm[r] = r;
    for (int j = j0 + tid; j < j1; j += TF_THREADS) spv[j - j0] = ipiv[j];  // (parallel global loads)
  }
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < SNJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) sC[(r0 + 8 * i + g) * LU_LDW + 8 * j + 2 * q + e] = acc[i][j][e];
  __syncthreads();
  if (tid == 0 && tp < 0)
    for (int j = j0; j < j1; ++j) {
      const int r = spv[j - j0] - 1;
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
}

// Block [c0, c0+ib) of the unit-lower solve on the register slab: its rows <- L_ss^{-1} rows
// (forward substitution), rows below -= L[rows, c0:c0+ib] * block rows (DMMA).  Lt: the tile
// holding L (explicit unit-lower copy or the factored tile itself; only r > c is read).
template <int MI>
__device__ __forceinline__ void lu_rows_block(double (&acc)[MI][SNJ][2], const double* Lt, int c0, int ib, int b,
                                              double* sm) {
  constexpr int RW = 8 * MI;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  const int r0 = warp * RW;
  const int c1 = c0 + ib;
  double* sU = sm;                // ib x LU_LDW
  double* sL = sU + 64 * LU_LDW;  // ib x (ib+1)
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
    sL[r * (ib + 1) + m] = (r > m) ? ldg_cg(Lt + (c0 + r) + (size_t)(c0 + m) * b) : 0.0;
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
  if (c1 < b && r0 + RW > c1) {
    for (int ks = 0; ks < ib / 4; ++ks) {
      double a[MI], bq[SNJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int row = r0 + 8 * i + g;
        a[i] = row >= c1 ? -Lt[row + (size_t)(c0 + 4 * ks + q) * b] : 0.0;
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

// GESSM item: 32 columns of C = A_kj <- L_kk^{-1} P_kk C.  LX = explicit unit-lower L_kk
// copy (b x b), ipiv = GETRF interchanges in [1, b] (LAPACK form, Z12).
template <int MI>
__device__ inline void gessm_reg(const Ctx& cx, const double* LX, const int* ipiv, double* C, int item,
                                 double* sm) {
  const int b = cx.b, ib = cx.ib;
  C += (size_t)item * NSR * b;
  double acc[MI][SNJ][2];
  slab_load<MI>(acc, C, b);
  lu_rows_permute<MI>(acc, ipiv, 0, b, b, sm);
  for (int c0 = 0; c0 < b; c0 += ib) lu_rows_block<MI>(acc, LX, c0, ib, b, sm);
  slab_store<MI>(acc, C, b);
}

// LU panel of one 32-column slab held as P (smem, b x 32, column-major, ld ldp) on entry and
// exit; registers during the factorization (warp w: rows [w*RW, (w+1)*RW), lane c: column c).
//   TS (TSTRF): pairwise pivoting of column jj between the top row jj of
//       UL (32 x 33: U of the slab's diagonal block above the diagonal, the L-strip block
//       below it, footnote PAPER.md:542-544) and all b rows of P; the top row wins ties
//       (first maximum in stacked order, Z11).  A swap exchanges the whole 32-entry row.
//       pivots: b + r + 1 (row r swapped in) or cs + jj + 1 (kept), Z13.
//   !TS (GETRF): partial pivoting over tile rows >= cs + jj of P (first
//       maximum), rows swapped over the slab's 32 columns (the caller applies them to the
//       other columns, Z12); pivots cs-relative rows + 1 in [1, b].
// Column jj: lane jj's local argmax -> barrier -> every warp merges in warp order -> the
// rows involved in the swap are published -> barrier -> swap, scaling by the pivot
// (division, as the oracle), rank-1 update of columns > jj.  Returns the first zero-pivot
// local column or -1.
template <int MI, bool TS>
__device__ inline int lu_panel(double* P, int ldp, int cs, int b, double* UL, int* piv, double* sm2) {
  constexpr int RW = 8 * MI;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = lane, r0w = warp * RW;
  double* amv = sm2;                                     // 16 warp maxima
  int* ami = reinterpret_cast<int*>(amv + 16);           // 16 warp argmax rows
  double* rowA = amv + 32;                               // 32: pivot row (pre-swap)
  double* rowB = rowA + 32;                              // 32: GETRF row cs + jj (pre-swap)
  double* xcol = rowB + 32;                              // 16 x RW: scaled column jj per warp
  double* xw = xcol + warp * RW;
  double p[RW];
#pragma unroll
  for (int k = 0; k < RW; ++k) p[k] = P[(r0w + k) + (size_t)c * ldp];
  int first_zero = -1;
  for (int jj = 0; jj < 32; ++jj) {
    const int cg = cs + jj;
    const int kcg = cg - r0w;
    // lane jj: first maximum of |x| over this warp's candidate rows
    // (pairwise trees over ordered halves: the left operand holds the lower rows, so taking
    //  the right one only when strictly larger keeps the first maximum)
    if (c == jj) {
      double v[RW];
      int id[RW];
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        v[k] = (TS || k >= kcg) ? fabs(p[k]) : -1.0;
        id[k] = (TS || k >= kcg) ? r0w + k : INT_MAX;
      }
#pragma unroll
      for (int st = 1; st < RW; st *= 2)
#pragma unroll
        for (int k = 0; k < RW; k += 2 * st)
          if (v[k + st] > v[k]) { v[k] = v[k + st]; id[k] = id[k + st]; }
      amv[warp] = v[0];
      ami[warp] = id[0];
    }
    __syncthreads();
    int pr;
    {
      double v[TF_WARPS];
      int id[TF_WARPS];
#pragma unroll
      for (int w = 0; w < TF_WARPS; ++w) { v[w] = amv[w]; id[w] = ami[w]; }
#pragma unroll
      for (int st = 1; st < TF_WARPS; st *= 2)
#pragma unroll
        for (int w = 0; w < TF_WARPS; w += 2 * st)
          if (v[w + st] > v[w]) { v[w] = v[w + st]; id[w] = id[w + st]; }
      double bv = TS ? fabs(UL[jj * 33 + jj]) : -1.0;
      pr = TS ? -1 : INT_MAX;
      if (v[0] > bv) { bv = v[0]; pr = id[0]; }
    }
    if (!TS && pr == INT_MAX) pr = cg;  // (no candidates cannot happen: row cg itself)
    const int kpr = pr - r0w;
    // publish the rows the swap exchanges (pre-swap values)
    if (pr >= 0 && kpr >= 0 && kpr < RW) {
      double tv = 0.0;
#pragma unroll
      for (int k = 0; k < RW; ++k)
        if (k == kpr) tv = p[k];
      rowA[c] = tv;
    }
    if (!TS && kcg >= 0 && kcg < RW) {
      double tv = 0.0;
#pragma unroll
      for (int k = 0; k < RW; ++k)
        if (k == kcg) tv = p[k];
      rowB[c] = tv;
    }
    __syncthreads();
    // the new top / pivot row, and the swap
    const double oldtop = TS ? UL[jj * 33 + c] : rowB[c];
    const double newtop = (TS && pr < 0) ? oldtop : rowA[c];
    const double u = __shfl_sync(0xffffffffu, newtop, jj);
    if (TS) {
      if (pr >= 0 && kpr >= 0 && kpr < RW) {
#pragma unroll
        for (int k = 0; k < RW; ++k)
          if (k == kpr) p[k] = oldtop;
      }
    } else if (pr != cg) {
      if (kpr >= 0 && kpr < RW) {
#pragma unroll
        for (int k = 0; k < RW; ++k)
          if (k == kpr) p[k] = oldtop;  // row pr <- row cg
      }
      if (kcg >= 0 && kcg < RW) {
#pragma unroll
        for (int k = 0; k < RW; ++k)
          if (k == kcg) p[k] = newtop;  // row cg <- row pr
      }
    }
    if (warp == 0) {
      if (TS) UL[jj * 33 + c] = newtop;
      if (c == 0) piv[jj] = TS ? (pr >= 0 ? b + pr + 1 : cg + 1) : pr + 1;
    }
    if (u != 0.0) {
      // multipliers of column jj (rows below the pivot), then the rank-1 update
      // (the divisions run one per lane, not serially on lane jj)
      __syncwarp();
      if (c == jj) {
#pragma unroll
        for (int k = 0; k < RW; ++k) xw[k] = (TS || k > kcg) ? p[k] : 0.0;
      }
      __syncwarp();
      if (c < RW) xw[c] = xw[c] / u;
      __syncwarp();
      if (c == jj) {
#pragma unroll
        for (int k = 0; k < RW; ++k)
          if (TS || k > kcg) p[k] = xw[k];
      }
      if (c > jj) {
#pragma unroll
        for (int k = 0; k < RW; k += 2) {
          const double2 x2 = *reinterpret_cast<const double2*>(xw + k);
          p[k] = fma(-x2.x, newtop, p[k]);
          p[k + 1] = fma(-x2.y, newtop, p[k + 1]);
        }
      }
    } else if (first_zero < 0) {
      first_zero = jj;
    }
  }
#pragma unroll
  for (int k = 0; k < RW; ++k) P[(r0w + k) + (size_t)c * ldp] = p[k];
  __syncthreads();
  return first_zero;
}

// TSTRF for ib = 32, left-looking over 32-column slabs: every finished
// block's pairwise swaps / unit-lower solve / update (lu_ts_apply), then the slab's panel.
// U: the diagonal tile (upper region only is touched), A: the tile below, Ls: L strip,
// ipiv: pivots (i,k).  Returns the first zero-pivot local column or -1.
template <int MI>
__device__ inline int tstrf_slab(const Ctx& cx, double* U, double* A, double* Ls, int* ipiv, double* sm) {
  const int b = cx.b, ib = cx.ib;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  constexpr int RW = 8 * MI;
  const int r0 = warp * RW;
  const int ldp = b + 1;
  int first_zero = -1;
  double acc[MI][SNJ][2];
  TF_LU_T0();
  for (int cs = 0; cs < b; cs += NSR) {
    slab_load<MI>(acc, A + (size_t)cs * b, b);
    for (int c0 = 0; c0 < cs; c0 += ib)
      lu_ts_apply<MI>(acc, U + c0 + (size_t)cs * b, A + (size_t)c0 * b, Ls + (size_t)c0 * ib, ipiv + c0, ib, b, sm);
    TF_LU_T(8);
    double* P = sm;
    double* UL = P + 32 * ldp;
    double* sm2 = UL + 32 * 33;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < SNJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) P[(r0 + 8 * i + g) + (size_t)(8 * j + 2 * q + e) * ldp] = acc[i][j][e];
    for (int e = tid; e < 32 * 32; e += TF_THREADS) {
      const int rr = e % 32, cc = e / 32;
      UL[rr * 33 + cc] = (rr <= cc) ? ldg_cg(U + (cs + rr) + (size_t)(cs + cc) * b) : 0.0;
    }
    __syncthreads();
    TF_LU_T(9);
    const int fz = lu_panel<MI, true>(P, ldp, cs, b, UL, ipiv + cs, sm2);
    if (fz >= 0 && first_zero < 0) first_zero = cs + fz;
    TF_LU_T(10);
    for (int e = tid; e < b * 32; e += TF_THREADS) {
      const int rr = e % b, cc = e / b;
      A[rr + (size_t)(cs + cc) * b] = P[rr + (size_t)cc * ldp];
    }
    for (int e = tid; e < 32 * 32; e += TF_THREADS) {
      const int rr = e % 32, cc = e / 32;
      if (rr <= cc) U[(cs + rr) + (size_t)(cs + cc) * b] = UL[rr * 33 + cc];
      Ls[(size_t)(cs + cc) * ib + rr] = rr > cc ? UL[rr * 33 + cc] : 0.0;
    }
    __syncthreads();
    TF_LU_T(11);
  }
  return first_zero;
}

// GETRF for ib = 32, left-looking over 32-column slabs: the slab gets all
// earlier row interchanges and block solves/updates, then its panel; the slab's interchanges
// are then applied to the columns on its left (LAPACK dgetrf semantics, Z12).  LX: explicit
// unit-lower copy written at the end.  Returns the first zero-pivot local column or -1.
template <int MI>
__device__ inline int getrf_slab(const Ctx& cx, double* A, int* ipiv, double* LX, double* sm) {
  const int b = cx.b, ib = cx.ib;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  constexpr int RW = 8 * MI;
  const int r0 = warp * RW;
  const int ldp = b + 1;
  int first_zero = -1;
  double acc[MI][SNJ][2];
  int tp = tid;  // running composition of the interchanges so far: row tid <- original row tp
  TF_LU_T0();
  for (int cs = 0; cs < b; cs += NSR) {
    slab_load<MI>(acc, A + (size_t)cs * b, b);
    if (cs > 0) {
      lu_rows_permute<MI>(acc, ipiv, 0, cs, b, sm, tp);
      TF_LU_T(0);
      for (int c0 = 0; c0 < cs; c0 += ib) lu_rows_block<MI>(acc, A, c0, ib, b, sm);
      TF_LU_T(1);
    }
    double* P = sm;
    double* sm2 = P + 32 * ldp;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < SNJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) P[(r0 + 8 * i + g) + (size_t)(8 * j + 2 * q + e) * ldp] = acc[i][j][e];
    __syncthreads();
    TF_LU_T(2);
    const int fz = lu_panel<MI, false>(P, ldp, cs, b, nullptr, ipiv + cs, sm2);
    if (fz >= 0 && first_zero < 0) first_zero = cs + fz;
    TF_LU_T(3);
    for (int e = tid; e < b * 32; e += TF_THREADS) {
      const int rr = e % b, cc = e / b;
      A[rr + (size_t)(cs + cc) * b] = P[rr + (size_t)cc * ldp];
    }
    __syncthreads();
    TF_LU_T(4);
    // this slab's interchanges on the columns to its left: composed once into the list of
    // rows that change (new row x <- old row src[x]), then gathered through shared memory
    if (cs > 0 || cs + NSR < b) {
      int* perm = reinterpret_cast<int*>(sm);  // rows [cs, b)
      int* chg = perm + 512;                   // changed rows (<= 64)
      int* src = chg + 64;
      int* nchg = src + 64;
      int* spv = nchg + 1;
      int* tpv = spv + 32;                     // b: the running composition
      double* buf = sm + 1024;                 // n x (column chunk of <= 256)
      for (int r = cs + tid; r < b; r += TF_THREADS) perm[r - cs] = r;
      if (tid < 32) spv[tid] = ipiv[cs + tid];
      if (tid < b) tpv[tid] = tp;
      if (tid == 0) *nchg = 0;
      __syncthreads();
      if (tid == 0)
        for (int j = cs; j < cs + 32; ++j) {
          const int r = spv[j - cs] - 1;
          const int t = perm[j - cs];
          perm[j - cs] = perm[r - cs];
          perm[r - cs] = t;
        }
      __syncthreads();
      if (tid >= cs && tid < b) tp = tpv[perm[tid - cs]];
      __syncthreads();  // perm / tpv are read above; the next slab's permute rewrites this smem
      if (cs > 0) {
      for (int x = cs + tid; x < b; x += TF_THREADS)
        if (perm[x - cs] != x) {
          const int k = atomicAdd(nchg, 1);
          chg[k] = x;
          src[k] = perm[x - cs];
        }
      __syncthreads();
      const int n = *nchg;
      for (int cc0 = 0; cc0 < cs; cc0 += 256) {
        const int nc = min(256, cs - cc0);
        for (int e = tid; e < n * nc; e += TF_THREADS) {
          const int x = e % n, cc = cc0 + e / n;
          buf[e] = A[src[x] + (size_t)cc * b];
        }
        __syncthreads();
        for (int e = tid; e < n * nc; e += TF_THREADS) {
          const int x = e % n, cc = cc0 + e / n;
          A[chg[x] + (size_t)cc * b] = buf[e];
        }
        __syncthreads();
      }
      }
    }
    TF_LU_T(5);
  }
  for (int e = tid; e < b * b; e += TF_THREADS) {
    const int r = e % b, cc = e / b;
    LX[e] = (r > cc) ? A[e] : (r == cc ? 1.0 : 0.0);
  }
  return first_zero;
}

}  // namespace tf
