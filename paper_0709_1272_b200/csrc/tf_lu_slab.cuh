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


// One inner block of the pairwise-pivoted update on a register slab (SSSSM step):
// [U_s; A] <- swaps of block s, U_s <- (I + Ls_s)^{-1} U_s, A -= L[:, s] U_s.
//   Us  : U rows c0.. of the slab columns, (m, c) at Us[m + c*b] (read, then written back)
//   Lc  : L columns of the block, (r, m) at Lc[r + m*b]
//   Lsb : Ls block s, (r, m) at Lsb[r + m*ldl];  pv: the block's IB pivots (1-based, [1, 2b])
// (IB may be a 32-column sub-block of a 64-column inner block: ldl = the strip's ib)
// The sequential pairwise swaps (top row jj <-> the bottom row pivot jj names, jj in order)
// are composed per 32 pivots with __match_any_sync: top row jj ends with the original
// content of the previous top row that named the same bottom row (or of that bottom row if
// none), and a named bottom row ends with the last top row that named it.  Each column then
// gathers in two shared-memory round trips instead of a 32-step dependent chain.
// Blocks applied in sequence double-buffer their inputs: while block s runs, the U rows,
// the L-strip block and the pivots of block s+1 land in the other buffer set by cp.async
// (LuBlk next), so only the first block of a sequence waits for its loads.
struct LuBlk {
  const double* Us;   // U rows of the block (slab columns), ld b
  const double* Lsb;  // L-strip block, ld ldl
  const int* pv;      // pivots
  int ib, ldl;
};
constexpr int LU_SETW = 64 * LU_LDW + 64 * 65 + 32;  // one buffer set: sU, sL, pivots (doubles)
__device__ __forceinline__ double* lu_set(double* sm, int buf) {
  // [sA | flag/srcT/lastS ints | set 0 | set 1]
  return sm + 64 * LU_LDW + 384 + buf * LU_SETW;
}
template <int IB>
__device__ __forceinline__ void lu_ts_prefetch(const LuBlk& nx, int b, double* set) {
  double* sU = set;
  double* sL = sU + 64 * LU_LDW;
  int* spv = reinterpret_cast<int*>(sL + 64 * 65);
  const int tid = threadIdx.x;
  for (int e = tid; e < IB * NSR; e += TF_THREADS) {
    const int m = e % IB, c = e / IB;
    cp_async8(sU + m * LU_LDW + c, nx.Us + m + (size_t)c * b, 8);
  }
  for (int e = tid; e < IB * IB; e += TF_THREADS) {
    const int r = e % IB, m = e / IB;
    const double* src = nx.Lsb + r + (size_t)m * nx.ldl;
    cp_async8(sL + r * (IB + 1) + m, r > m ? src : nx.Lsb, r > m ? 8 : 0);  // zero-fill r <= m
  }
  if (tid < IB) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(spv + tid)), "l"(nx.pv + tid));
  cp_async_commit();
}

template <int MI, int IB>
__device__ __forceinline__ void lu_ts_apply_t(double (&acc)[MI][SNJ][2], double* Us, const double* Lc,
                                              const LuBlk& cur, int b, double* sm, int buf, bool pre,
                                              const LuBlk* nx) {
  constexpr int RW = 8 * MI;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  const int r0 = warp * RW;
  double* sA = sm;                              // IB slots x LU_LDW: the A rows the pivots name
  int* flag = reinterpret_cast<int*>(sA + 64 * LU_LDW);  // b: slot of bottom row r (INT_MAX = none)
  int* srcT = flag + 512;                       // top row P <- top row srcT (< 64) or slot srcT - 64
  int* lastS = srcT + 64;                       // [half][slot]: the slot <- top row lastS (-1: kept)
  double* sU = lu_set(sm, buf);                 // IB x LU_LDW: U_s
  double* sL = sU + 64 * LU_LDW;                // IB x (IB+1): L(r, m), r > m
  int* spv = reinterpret_cast<int*>(sL + 64 * 65);  // IB pivots of the block
  // the L columns of the update, in flight from the start (they are this block's own
  // results, L2-resident): MI * IB/4 values per thread
  constexpr int NPRE = (MI * IB / 4 <= 16) ? IB / 4 : 0;
  double la[NPRE > 0 ? NPRE : 1][MI];
  TF_LU_T0();
#pragma unroll
  for (int ks = 0; ks < NPRE; ++ks)
#pragma unroll
    for (int i = 0; i < MI; ++i) la[ks][i] = -Lc[(r0 + 8 * i + g) + (size_t)(4 * ks + q) * b];
  for (int r = tid; r < b; r += TF_THREADS) flag[r] = INT_MAX;
  // this block's inputs: requested now, or by the previous block's call (the only cp.async
  // group in flight at this point; the next block's is issued after the solve below)
  if (!pre) lu_ts_prefetch<IB>(cur, b, sU);
  cp_async_wait<0>();
  __syncthreads();
  TF_LU_T(16);
  if (tid < IB) {
    const int v = spv[tid];
    if (v > b) atomicMin(&flag[v - b - 1], tid);  // slot = first pivot naming the row
  }
  __syncthreads();
  // compose each half's swaps (warp h: pivots 32h .. 32h + 31)
  if (warp < IB / 32) {
    const int P = 32 * warp + lane;
    const int v = spv[P];
    const int f = v > b ? flag[v - b - 1] : -1;
    const unsigned m = __match_any_sync(0xffffffffu, f >= 0 ? f : 1000 + P);
    const unsigned below = m & ((1u << lane) - 1u);
    const int prev = below ? 31 - __clz(below) : -1;
    srcT[P] = f < 0 ? P : (prev >= 0 ? 32 * warp + prev : 64 + f);
    lastS[warp * 64 + lane] = -1;
    lastS[warp * 64 + 32 + lane] = -1;
    __syncwarp();
    if (f >= 0 && (m >> lane) == 1u) lastS[warp * 64 + f] = P;
  }
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
  TF_LU_T(17);
  // the composed swaps (16 lanes per column), then the unit-lower solve (per column)
  {
    const int c = tid >> 4, l = tid & 15;
#pragma unroll
    for (int h = 0; h < IB / 32; ++h) {
      double vt[2], vs[IB / 16];
      int ls[IB / 16];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int sr = srcT[32 * h + l + 16 * u];
        vt[u] = sr < 64 ? sU[sr * LU_LDW + c] : sA[(sr - 64) * LU_LDW + c];
      }
#pragma unroll
      for (int u = 0; u < IB / 16; ++u) {
        const int f = l + 16 * u;
        ls[u] = lastS[h * 64 + f];
        vs[u] = ls[u] >= 0 ? sU[ls[u] * LU_LDW + c] : 0.0;
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 2; ++u) sU[(32 * h + l + 16 * u) * LU_LDW + c] = vt[u];
#pragma unroll
      for (int u = 0; u < IB / 16; ++u)
        if (ls[u] >= 0) sA[(l + 16 * u) * LU_LDW + c] = vs[u];
      __syncwarp();
    }
    lu_block_solve(sU, sL, IB);
  }
  __syncthreads();
  TF_LU_T(18);
  // the next block's inputs into the other buffer set while this one finishes
  if (nx) {
    if (nx->ib == 32) lu_ts_prefetch<32>(*nx, b, lu_set(sm, buf ^ 1));
    else lu_ts_prefetch<64>(*nx, b, lu_set(sm, buf ^ 1));
  }
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int f = flag[r0 + 8 * i + g];
    if (f != INT_MAX)
#pragma unroll
      for (int j = 0; j < SNJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) acc[i][j][e] = sA[f * LU_LDW + 8 * j + 2 * q + e];
  }
  for (int e = tid; e < IB * NSR; e += TF_THREADS) {
    const int m = e % IB, c = e / IB;
    Us[m + (size_t)c * b] = sU[m * LU_LDW + c];
  }
  TF_LU_T(19);
  // A -= L[:, block] U_s (L operand one k-step ahead when it is not preloaded)
  double an[MI];
  if (!NPRE) {
#pragma unroll
    for (int i = 0; i < MI; ++i) an[i] = Lc[(r0 + 8 * i + g) + (size_t)q * b];
  }
#pragma unroll
  for (int ks = 0; ks < IB / 4; ++ks) {
    double a[MI], bq[SNJ];
    // (the sign folds into the DMMA operand modifier; no DADD on the shared FP64 pipe)
#pragma unroll
    for (int i = 0; i < MI; ++i) a[i] = NPRE ? la[NPRE ? ks : 0][i] : -an[i];
    if (!NPRE && ks + 1 < IB / 4) {
#pragma unroll
      for (int i = 0; i < MI; ++i) an[i] = Lc[(r0 + 8 * i + g) + (size_t)(4 * (ks + 1) + q) * b];
    }
#pragma unroll
    for (int j = 0; j < SNJ; ++j) bq[j] = sU[(4 * ks + q) * LU_LDW + 8 * j + g];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < SNJ; ++j) dmma(acc[i][j], a[i], bq[j]);
  }
  __syncthreads();
  TF_LU_T(20);
}

// Apply `cur` (buffer set `buf`; pre = its inputs were already requested by the previous
// call), prefetching `nx` (may be null) into the other set.  Returns the next buffer set.
template <int MI>
__device__ __forceinline__ int lu_ts_apply(double (&acc)[MI][SNJ][2], double* Us, const double* Lc,
                                           const LuBlk& cur, int b, double* sm, int buf, bool pre,
                                           const LuBlk* nx) {
  if (cur.ib == 32) lu_ts_apply_t<MI, 32>(acc, Us, Lc, cur, b, sm, buf, pre, nx);
  else lu_ts_apply_t<MI, 64>(acc, Us, Lc, cur, b, sm, buf, pre, nx);
  return buf ^ 1;
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
  int buf = 0;
  for (int c0 = 0; c0 < b; c0 += ib) {
    const LuBlk cur{U + c0, Ls + (size_t)c0 * ib, ipiv + c0, ib, ib};
    const LuBlk nxt{U + c0 + ib, Ls + (size_t)(c0 + ib) * ib, ipiv + c0 + ib, ib, ib};
    buf = lu_ts_apply<MI>(acc, U + c0, L + (size_t)c0 * b, cur, b, sm, buf, c0 > 0, c0 + ib < b ? &nxt : nullptr);
  }
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

// Block [c0, c0+IB) of the unit-lower solve on the register slab: its rows <- L_ss^{-1} rows
// (forward substitution), rows below -= L[rows, c0:c0+IB] * block rows (DMMA).  Lt: the tile
// holding L (explicit unit-lower copy or the factored tile itself; only r > c is read).
// The update's L operand is loaded at the start (in flight during the solve) when it fits.
#ifndef TF_RB_PRE
#define TF_RB_PRE 8
#endif
template <int MI, int IB>
__device__ __forceinline__ void lu_rows_block_t(double (&acc)[MI][SNJ][2], const double* Lt, int c0, int b,
                                                double* sm) {
  constexpr int RW = 8 * MI;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  const int r0 = warp * RW;
  const int c1 = c0 + IB;
  double* sU = sm;                // IB x LU_LDW
  double* sL = sU + 64 * LU_LDW;  // IB x (IB+1)
  const bool upd = c1 < b && r0 + RW > c1;
  constexpr int NPRE = (MI * IB / 4 <= TF_RB_PRE) ? IB / 4 : 0;
  double la[NPRE > 0 ? NPRE : 1][MI];
  if (upd) {
#pragma unroll
    for (int ks = 0; ks < NPRE; ++ks)
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int row = r0 + 8 * i + g;
        la[ks][i] = row >= c1 ? -Lt[row + (size_t)(c0 + 4 * ks + q) * b] : 0.0;
      }
  }
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int row = r0 + 8 * i + g;
    if (row >= c0 && row < c1)
#pragma unroll
      for (int j = 0; j < SNJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) sU[(row - c0) * LU_LDW + 8 * j + 2 * q + e] = acc[i][j][e];
  }
  for (int e = tid; e < IB * IB; e += TF_THREADS) {
    const int r = e % IB, m = e / IB;
    sL[r * (IB + 1) + m] = (r > m) ? ldg_cg(Lt + (c0 + r) + (size_t)(c0 + m) * b) : 0.0;
  }
  __syncthreads();
  lu_block_solve(sU, sL, IB);
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
  if (upd) {
#pragma unroll
    for (int ks = 0; ks < IB / 4; ++ks) {
      double a[MI], bq[SNJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int row = r0 + 8 * i + g;
        a[i] = NPRE ? la[NPRE ? ks : 0][i] : (row >= c1 ? -Lt[row + (size_t)(c0 + 4 * ks + q) * b] : 0.0);
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

template <int MI>
__device__ __forceinline__ void lu_rows_block(double (&acc)[MI][SNJ][2], const double* Lt, int c0, int ib, int b,
                                              double* sm) {
  if (ib == 32) lu_rows_block_t<MI, 32>(acc, Lt, c0, b, sm);
  else lu_rows_block_t<MI, 64>(acc, Lt, c0, b, sm);
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

__device__ __forceinline__ void bar_named(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void warp_first_max(double v, int idx, double& bv, int& bi) {
  // v >= 0 (fabs), idx = key (INT_MAX: no candidate).  Largest v, then smallest idx.
  const unsigned hi = (unsigned)__double2hiint(v), lo = (unsigned)__double2loint(v);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  bi = __reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? idx : INT_MAX);
  bv = __hiloint2double((int)mhi, (int)mlo);
}

constexpr int ULD = 34;  // row stride of the TSTRF top block UL (16-byte aligned rows)

// LU panel of one 32-column slab held as P (smem, b x 32, column-major, ld ldp) on entry and
// exit.  Row-per-thread: thread t < b keeps row t of the slab (32 doubles) in registers, so
// the pivot search of a column is a reduction over threads and the rank-1 update is
// 31 - jj FMAs per thread with the pivot row broadcast from smem.
//   TS (TSTRF): pairwise pivoting of column jj between the top row jj of
//       UL (32 x ULD: U of the slab's diagonal block above the diagonal, the L-strip block
//       below it, footnote PAPER.md:542-544) and all b rows of P; the top row wins ties
//       (first maximum in stacked order, Z11).  A swap exchanges the whole 32-entry row.
//       pivots: b + r + 1 (row r swapped in) or cs + jj + 1 (kept), Z13.
//   !TS (GETRF): partial pivoting over tile rows >= cs + jj of P (first
//       maximum), rows interchanged over the slab's 32 columns (the caller applies them to
//       the other columns, Z12); pivots cs-relative rows + 1 in [1, b].  The interchanges
//       are applied lazily: thread t tracks the row position `pos` its registers hold (an
//       interchange swaps two positions, no data moves), candidates and ties are decided on
//       positions (first maximum = smallest position), and rows land at their final
//       positions when the panel is written back.
// Column jj, TWO barriers over the warps that own rows (named barrier; the other warps
// skip the panel): (A) every warp publishes its candidate (max |x|, smallest position
// among the maxima, and that row's reciprocal, formed while the reductions run) with one
// lane's stores; after A every warp merges the candidates the same way, so all threads
// know the pivot row, and only the pivot row's thread publishes its columns jj..31;
// (B) then division (x r with the division's own correction, = x / upiv bitwise), the
// update of column jj + 1 first, column jj + 1's warp candidates, and the rest of the
// rank-1 update while the reductions run.  (Measured: a barrier after s one-lane 128-bit
// shared stores per warp costs ~5.5 cycles per store instruction in the CTA, so the
// round-1 design — every warp's candidate publishing its whole row and one barrier —
// spent ~0.8-1.4k cycles per column on the store drain; tools/lat_stsbar.cu.)
// Returns the first zero-pivot local column or -1.
template <int MI, bool TS>
__device__ inline int lu_panel(double* P, int ldp, int cs, int b, double* UL, int* piv, double* sm2, int nopiv) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwa = (b + 31) >> 5;                         // warps that own rows
  const bool own = tid < b;
  double2* sv = reinterpret_cast<double2*>(sm2);         // [2][16] {max |x|, reciprocal}
  int* sk = reinterpret_cast<int*>(sm2 + 64);            // [2][16] key = position << 4 | warp
  double* urow = sm2 + 80;                               // [2][32] the pivot row
  int* fzp = reinterpret_cast<int*>(sm2 + 144);
  double x[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) x[c] = own ? P[tid + (size_t)c * ldp] : 0.0;
  int pos = tid;
  int first_zero = -1;
  // the warp's candidate for column jj -> slot (par, warp); GENP (nopiv): GETRF's only
  // candidate is position cs + jj, TSTRF keeps the top row
  auto candidate = [&](int jj, int par) {
    const bool cand = own && (TS ? !nopiv : (nopiv ? pos == cs + jj : pos >= cs + jj));
    const int key = cand ? (pos << 4 | warp) : INT_MAX;
    const double rr = rcp_newton(x[jj]);
    double wv;
    int wk;
    warp_first_max(cand ? fabs(x[jj]) : 0.0, key, wv, wk);
    if (wk == INT_MAX ? lane == 0 : key == wk) {
      sv[par * 16 + warp] = make_double2(wv, rr);
      sk[par * 16 + warp] = wk;
    }
  };
  TF_LU_T0();
  if (warp < nwa) {
    candidate(0, 0);
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      const int par = jj & 1;
      const int cg = cs + jj;
      // (TSTRF) the top candidate and its reciprocal, before A (the winner rewrites UL row
      // jj after B; nothing else writes it)
      const double top = TS ? UL[jj * ULD + jj] : 0.0;
      const double rtop = TS ? rcp_newton(top) : 0.0;
      TF_LU_T(12);
      bar_named(1, nwa * 32);
      TF_LU_T(13);
      double2 v = make_double2(0.0, 0.0);
      int k = INT_MAX;
      if (lane < nwa) {
        v = sv[par * 16 + lane];
        k = sk[par * 16 + lane];
      }
      double bv;
      int kmin;
      warp_first_max(v.x, k, bv, kmin);
      double r = __shfl_sync(0xffffffffu, v.y, kmin & 15);
      int pr = kmin == INT_MAX ? -1 : kmin >> 4;         // GETRF: a candidate always exists
      if (TS && !(bv > fabs(top))) {                     // the top row wins ties
        pr = -1;
        r = rtop;
      }
      const bool win = TS ? (pr >= 0 && tid == pr) : (pos == pr);
      if (win) {
#pragma unroll
        for (int c = jj & ~1; c < 32; c += 2)
          *reinterpret_cast<double2*>(urow + par * 32 + c) = make_double2(x[c], x[c + 1]);
      }
      TF_LU_T(14);
      bar_named(1, nwa * 32);
      const double* u = (TS && pr < 0) ? UL + jj * ULD : urow + par * 32;
      if (tid == 0) piv[jj] = TS ? (pr >= 0 ? b + pr + 1 : cg + 1) : pr + 1;
      if (TS) {
        if (win) {  // row pr <-> top row jj (the whole 32-entry row)
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const double2 t = *reinterpret_cast<const double2*>(UL + jj * ULD + c);
            *reinterpret_cast<double2*>(UL + jj * ULD + c) = make_double2(x[c], x[c + 1]);
            x[c] = t.x;
            x[c + 1] = t.y;
          }
        }
      } else if (win) {
        pos = cg;
      } else if (pos == cg) {
        pos = pr;
      }
      const double upiv = u[jj];
      const bool elim = own && (TS || pos > cg) && upiv != 0.0;
      double l = 0.0;
      if (elim) {
        l = div_rcp(x[jj], upiv, r);
        x[jj] = l;
        if (jj < 31) x[jj + 1] = fma(-l, u[jj + 1], x[jj + 1]);
      }
      if (upiv == 0.0 && first_zero < 0) first_zero = jj;
      if (jj < 31) {
        candidate(jj + 1, par ^ 1);
        if (elim) {
#pragma unroll
          for (int c = jj + 2; c < 32; ++c) x[c] = fma(-l, u[c], x[c]);
        }
      }
      TF_LU_T(15);
    }
  }
  if (own) {
#pragma unroll
    for (int c = 0; c < 32; ++c) P[pos + (size_t)c * ldp] = x[c];
  }
  // warps without rows skipped the pivot tests: every thread takes thread 0's first_zero
  if (tid == 0) *fzp = first_zero;
  __syncthreads();
  first_zero = *fzp;
  __syncthreads();
  return first_zero;
}


// TSTRF for ib in {32, 64}, left-looking over 32-column slabs: every
// finished inner block's pairwise swaps / unit-lower solve / update (lu_ts_apply), then the
// slab's panel.  With ib = 64 an inner block is two slabs: the second slab first applies
// the first slab as a 32-column sub-block (swaps of its pivots, (I + Ls_11)^{-1} on its top
// rows, the rank-32 update), and after its own panel moves the first slab's multipliers of
// the rows it swapped in into the L strip (footnote PAPER.md:542-544: a pivot of column j
// exchanges the Ls row j - c0 with the bottom row over columns [c0, j); deferred to after
// the panel, in pivot order, since nothing else touches those columns meanwhile).
// U: the diagonal tile (upper region only is touched), A: the tile below, Ls: L strip,
// ipiv: pivots (i,k).  Returns the first zero-pivot local column or -1.
template <int MI>
// Slabs [c_begin, c_end) only (the slab-level DAG's TSTRF slab tasks).
// blk_lo / blk_hi / panel: as qr_slab (the slab-level graph's TSTRF apply tasks).
__device__ inline int tstrf_slab(const Ctx& cx, double* U, double* A, double* Ls, int* ipiv, int c_begin, int c_end,
                                 double* sm, int blk_lo = 0, int blk_hi = INT_MAX, bool panel = true) {
  const int b = cx.b, ib = cx.ib;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  constexpr int RW = 8 * MI;
  const int r0 = warp * RW;
  const int ldp = b + 1;
  int first_zero = -1;
  double acc[MI][SNJ][2];
  TF_LU_T0();
  for (int cs = c_begin; cs < c_end; cs += NSR) {
    const int s0 = cs - cs % ib, off = cs - s0;  // this slab's inner block and its offset in it
    slab_load<MI>(acc, A + (size_t)cs * b, b);
    {
      // the finished inner blocks, then (second slab of a 64-block) the block's first slab
      // as a 32-column sub-block; each block's inputs prefetched during the previous one
      int buf = 0;
      const int nfull = s0 / ib;
      const int xlo = blk_lo < nfull ? blk_lo : nfull;
      const int xhi = panel ? nfull + (off ? 1 : 0) : (blk_hi < nfull ? blk_hi : nfull);
      auto blk = [&](int x) {
        const int c0 = x < nfull ? x * ib : s0;
        return LuBlk{U + c0 + (size_t)cs * b, Ls + (size_t)c0 * ib, ipiv + c0, x < nfull ? ib : NSR, ib};
      };
      for (int x = xlo; x < xhi; ++x) {
        const LuBlk cur = blk(x), nxt = blk(x + 1 < xhi ? x + 1 : x);
        const int c0 = x < nfull ? x * ib : s0;
        buf = lu_ts_apply<MI>(acc, U + c0 + (size_t)cs * b, A + (size_t)c0 * b, cur, b, sm, buf, x > xlo,
                              x + 1 < xhi ? &nxt : nullptr);
      }
    }
    if (!panel) {
      slab_store<MI>(acc, A + (size_t)cs * b, b);
      __syncthreads();
      continue;
    }
    TF_LU_T(8);
    double* P = sm;
    double* UL = P + 32 * ldp;
    double* sm2 = UL + 32 * ULD;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < SNJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) P[(r0 + 8 * i + g) + (size_t)(8 * j + 2 * q + e) * ldp] = acc[i][j][e];
    for (int e = tid; e < 32 * 32; e += TF_THREADS) {
      const int rr = e % 32, cc = e / 32;
      UL[rr * ULD + cc] = (rr <= cc) ? ldg_cg(U + (cs + rr) + (size_t)(cs + cc) * b) : 0.0;
    }
    __syncthreads();
    TF_LU_T(9);
    const int fz = lu_panel<MI, true>(P, ldp, cs, b, UL, ipiv + cs, sm2, cx.nopiv);
    if (fz >= 0 && first_zero < 0) first_zero = cs + fz;
    TF_LU_T(10);
    for (int e = tid; e < b * 32; e += TF_THREADS) {
      const int rr = e % b, cc = e / b;
      A[rr + (size_t)(cs + cc) * b] = P[rr + (size_t)cc * ldp];
    }
    for (int e = tid; e < 32 * 32; e += TF_THREADS) {
      const int rr = e % 32, cc = e / 32;
      if (rr <= cc) U[(cs + rr) + (size_t)(cs + cc) * b] = UL[rr * ULD + cc];
      Ls[(size_t)(cs + cc) * ib + off + rr] = rr > cc ? UL[rr * ULD + cc] : 0.0;
      if (ib == 2 * NSR) Ls[(size_t)(cs + cc) * ib + (NSR - off) + rr] = 0.0;  // the other half's rows
    }
    __syncthreads();
    if (off && tid < NSR) {
      // first slab's multiplier rows swapped in by this slab's pivots -> L-strip rows
      // (one thread per column s0 + tid, pivots in order)
      const int c = s0 + tid;
      for (int jj = 0; jj < NSR; ++jj) {
        const int pv = ipiv[cs + jj];
        if (pv > b) {
          double* lp = Ls + (size_t)c * ib + off + jj;
          double* ap = A + (pv - b - 1) + (size_t)c * b;
          const double t = *lp;
          *lp = *ap;
          *ap = t;
        }
      }
    }
    __syncthreads();
    TF_LU_T(11);
  }
  return first_zero;
}

// GETRF for ib in {32, 64}, left-looking over 32-column slabs: the slab gets all
// earlier row interchanges and block solves/updates, then its panel; the slab's interchanges
// are then applied to the columns on its left (LAPACK dgetrf semantics, Z12).  LX: explicit
// unit-lower copy written at the end.  Returns the first zero-pivot local column or -1.
template <int MI>
// Slabs [c_begin, c_end) only (the slab-level DAG's GETRF slab tasks): between slab tasks the
// running composition of the interchanges (tp) is parked in the first b ints of LX, which is
// written only after the last slab.
__device__ inline int getrf_slab(const Ctx& cx, double* A, int* ipiv, double* LX, int c_begin, int c_end,
                                 double* sm) {
  const int b = cx.b, ib = cx.ib;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  constexpr int RW = 8 * MI;
  const int r0 = warp * RW;
  const int ldp = b + 1;
  int first_zero = -1;
  double acc[MI][SNJ][2];
  int* tp_park = reinterpret_cast<int*>(LX);
  // running composition of the interchanges so far: row tid <- original row tp
  int tp = (c_begin > 0 && tid < b) ? ld_cg_int(tp_park + tid) : tid;
  TF_LU_T0();
  for (int cs = c_begin; cs < c_end; cs += NSR) {
    slab_load<MI>(acc, A + (size_t)cs * b, b);
    if (cs > 0) {
      lu_rows_permute<MI>(acc, ipiv, 0, cs, b, sm, tp);
      TF_LU_T(0);
      // unit-lower block solves / updates by 32-column blocks whatever ib is (the blocking
      // of the forward substitution does not change it beyond rounding)
      for (int c0 = 0; c0 < cs; c0 += NSR) lu_rows_block<MI>(acc, A, c0, NSR, b, sm);
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
    const int fz = lu_panel<MI, false>(P, ldp, cs, b, nullptr, ipiv + cs, sm2, cx.nopiv);
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
  if (c_end < b) {
    if (tid < b) tp_park[tid] = tp;
    return first_zero;
  }
  __syncthreads();  // (every thread's parked tp was read before LX is overwritten)
  for (int e = tid; e < b * b; e += TF_THREADS) {
    const int r = e % b, cc = e / b;
    LX[e] = (r > cc) ? A[e] : (r == cc ? 1.0 : 0.0);
  }
  return first_zero;
}

}  // namespace tf
