// tf_kernels.cuh — the eleven tile kernels of Algorithms 1-3 as CTA-wide device
// functions (512 threads, one work item each), called by the persistent scheduler
// (tf_lib.cu) and by the per-kernel test launcher tk_run.
//
//   Cholesky:  POTRF, TRSM, SYRK (DGSMM i=j), GEMM (DGSMM i>j)
//   QR:  GEQRT, LARFB, TSQRT, SSRFB   (inner block ib, §3.2.3)
//   LU:  GETRF, GESSM, TSTRF, SSSSM   (L strips)
//
// Semantics follow SURVEY.md §8(c) C1-C3 (the readings adopted in DESIGN.md §3); the
// arithmetic is blocked for the hardware (DMMA engine for every dense update, warp-level
// panels), so results agree with the oracle to rounding, and bitwise on the exact pins.
//
// Work items: update tasks are split so several CTAs work on one task — TRSM by
// 128-row blocks, SYRK/GEMM by 128x128 output sub-tiles, LARFB/SSRFB/GESSM/SSSSM by
// column slabs of NS columns.  Panel tasks (POTRF/GEQRT/TSQRT/GETRF/TSTRF) are one item.
//
// Memory-model notes: tile data is read with L2-only loads (cp.async.cg / ld.global.cg)
// or through shared memory; tasks that write only the R/U ("up") region of a diagonal
// tile store element by element inside that region, never over V/L.
#pragma once
#include <climits>
#include "tf_gemm.cuh"
#include "tf_sched.h"

namespace tf {

constexpr int NB = 32;               // column block of the in-CTA POTRF / TRSM solves

struct Ctx {
  int b, ib;
  double* scratch;  // this CTA's global scratch (>= 2*ib*b + 64 doubles)
  int* info;        // INT_MAX = no failure; atomicMin of the 1-based global column
  int* abort_flag;  // set on Cholesky failure: the scheduler stops handing out work
  int nopiv;        // LU without pivoting (GENP): every pivot is kept
};

// Kernel variants (register-slab kernel at one tile size, or the reference-blocked path):
// in the persistent build (TF_SPLIT_ITEMS) each variant is a separate function with its own
// register allocation; elsewhere (tk_run, tools) they inline.  A variant re-declares the
// dynamic shared memory so the shared address space stays known inside it.
#ifdef TF_SPLIT_ITEMS
#define TF_VARIANT __device__ __noinline__
#else
#define TF_VARIANT __device__ __forceinline__
#endif
#define TF_DSM_DECL extern __shared__ __align__(16) double dsm[]
#define TF_DEF_VARIANT(name, fn, params, args) \
  template <int MI>                             \
  TF_VARIANT void name params {                 \
    TF_DSM_DECL;                                \
    fn<MI> args;                                \
  }
#define TF_DEF_VARIANT_RET(name, fn, params, args) \
  template <int MI>                                 \
  TF_VARIANT int name params {                      \
    TF_DSM_DECL;                                    \
    return fn<MI> args;                             \
  }
#define TF_DEF_REF(name, fn, params, args) \
  TF_VARIANT void name params {             \
    TF_DSM_DECL;                            \
    fn args;                                \
  }
#define TF_DEF_REF_RET(name, fn, params, args) \
  TF_VARIANT int name params {                  \
    TF_DSM_DECL;                                \
    return fn args;                             \
  }

using GemmNT128 = Gemm<128, 128, 4, 4, false, false>;
using GemmNT32 = Gemm<128, 32, 8, 2, false, false>;
using GemmW64 = Gemm<64, 64, 4, 4, true, true>;
using GemmW32 = Gemm<32, 128, 2, 8, true, true>;
using GemmUpd = Gemm<128, 64, 4, 4, false, true>;

// C(M x N, ldc) -= Aop * Bop over tiles of the update engine (A m-contig, B k-major).
__device__ inline void update_mn(double* sm, double* C, int ldc, const double* A, int lda, const double* B,
                                 int ldb, int M, int N, int K) {
  for (int n0 = 0; n0 < N; n0 += 64)
    for (int m0 = 0; m0 < M; m0 += 128) {
      GemmUpd g;
      g.zero();
      const int mm = min(128, M - m0), nn = min(64, N - n0);
      g.run(sm, A + m0, lda, B + (size_t)n0 * ldb, ldb, mm, nn, K);
      sub_store(g, C + m0 + (size_t)n0 * ldc, ldc, mm, nn);
    }
}

// W(M x N, ld ldw) = Aop^T-style product with both operands k-major (+ optional addend
// R(M x N, ldr) read from global), written to W.  Used for W = V^T C (+ R).
__device__ inline void w_product(double* sm, double* W, int ldw, const double* A, int lda, const double* B,
                                 int ldb, int M, int N, int K, const double* R, int ldr) {
  if (M <= 32) {
    for (int n0 = 0; n0 < N; n0 += 128) {
      GemmW32 g;
      g.zero();
      const int nn = min(128, N - n0);
      g.run(sm, A, lda, B + (size_t)n0 * ldb, ldb, M, nn, K);
      g.for_each(M, nn, [&](int r, int c, double v) {
        const int cc = n0 + c;
        W[r + (size_t)cc * ldw] = R ? v + ldg_cg(R + r + (size_t)cc * ldr) : v;
      });
    }
  } else {
    for (int m0 = 0; m0 < M; m0 += 64)
      for (int n0 = 0; n0 < N; n0 += 64) {
        GemmW64 g;
        g.zero();
        const int mm = min(64, M - m0), nn = min(64, N - n0);
        g.run(sm, A + (size_t)m0 * lda, lda, B + (size_t)n0 * ldb, ldb, mm, nn, K);
        g.for_each(mm, nn, [&](int r, int c, double v) {
          const int rr = m0 + r, cc = n0 + c;
          W[rr + (size_t)cc * ldw] = R ? v + ldg_cg(R + rr + (size_t)cc * ldr) : v;
        });
      }
  }
  __syncthreads();
}

// W2 = T^T W for an upper-triangular ib x ib T (smem, ld ldt): W2[m][n] = sum_{q<=m} T[q][m] W[q][n].
__device__ inline void apply_tt(const double* sT, int ldt, const double* W, double* W2, int ib, int N) {
  for (int e = threadIdx.x; e < ib * N; e += TF_THREADS) {
    const int m = e % ib, n = e / ib;
    double s = 0.0;
    for (int q = 0; q <= m; ++q) s += sT[q + m * ldt] * W[q + (size_t)n * ib];
    W2[m + (size_t)n * ib] = s;
  }
  __syncthreads();
}

// Load the T_s block (ib x ib) of strip Tst into shared memory (ld ib).
__device__ inline void load_ts(double* sT, const double* Tst, int ib, int c0) {
  for (int e = threadIdx.x; e < ib * ib; e += TF_THREADS) sT[e] = ldg_cg(Tst + (size_t)c0 * ib + e);
  __syncthreads();
}

// ====================================================================================
// Cholesky (C1)
// ====================================================================================

// In-place Cholesky of the nb x nb lower block D (smem, ld NB+1) by warp 0 (DPOTF2,
// PAPER.md:260-267).  Returns -1 or the failing local column.
// nb = NB: right-looking, fully unrolled; lane i keeps row i in registers.  After column j
// every lane applies the rank-1 update x_i[c] -= L[i][j] L[c][j] (c > j) with L[c][j] read
// back from shared memory (broadcast loads), while lane j+1 forms the next pivot
// x_{j+1}[j+1] - L[j+1][j]^2 at once and shuffles it: the per-column critical path is one
// shuffle, one rsqrt, one multiply and one FMA (175 cycles per column against 262 for the
// left-looking form with four partial sums, tools/chol_bench.cu).  The subtractions of each
// element happen in the same order (m = 0, 1, ..., j-1) as the oracle's DPOTF2 dot products.
// No early exit and no divergent branches: the first failing column is recorded.
// (A register-resident variant with the multipliers by shuffles was measured slower: 496
// shuffles issue from one warp; potrf b=128 63 -> 136 us.)
__device__ inline int chol_diag_block(double* D, int nb, int* sflag) {
  if (nb == NB) {
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
        const double l = (lane == j ? d : x[j]) * r;  // L_jj = d / sqrt(d), L_ij = x_i[j] / sqrt(d)
        if (lane >= j) D[lane + j * (NB + 1)] = l;
        if (lane == j) D[NB + j * (NB + 1)] = r;  // padding row: reciprocal of L_jj for row_solve
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
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int fail = -1;
    for (int j = 0; j < nb; ++j) {
      double s = 0.0;
      if (lane >= j && lane < nb) {
        // two interleaved partial sums halve the dependent FMA chain (rounding order only)
        double s0 = D[lane + j * (NB + 1)], s1 = 0.0;
        int m = 0;
        for (; m + 1 < j; m += 2) {
          s0 -= D[lane + m * (NB + 1)] * D[j + m * (NB + 1)];
          s1 -= D[lane + (m + 1) * (NB + 1)] * D[j + (m + 1) * (NB + 1)];
        }
        if (m < j) s0 -= D[lane + m * (NB + 1)] * D[j + m * (NB + 1)];
        s = s0 + s1;
      }
      const double d = __shfl_sync(0xffffffffu, s, j);
      if (!(d > 0.0)) { fail = j; break; }
      // 1/sqrt once per column: L_jj = d * r, L_rj = s * r (no division in the chain)
      const double r = rsqrt(d);
      if (lane == j) {
        D[j + j * (NB + 1)] = d * r;
        D[NB + j * (NB + 1)] = r;  // padding row: reciprocal of L_jj for row_solve
      } else if (lane > j && lane < nb) {
        D[lane + j * (NB + 1)] = s * r;
      }
      __syncwarp();
    }
    if (lane == 0) *sflag = fail;
  }
  __syncthreads();
  return *sflag;
}

// X[r, 0:nb] <- X[r, 0:nb] * D^{-T} for rows r in [0, rows) (X global, ld ldx), D the
// lower nb x nb block in smem (ld NB+1).  Row-parallel; right-looking inside a row:
// X[r,c] = (A[r,c] - sum_{m<c} X[r,m] D[c,m]) / D[c,c] (DTRSM).
__device__ inline void row_solve(double* X, int ldx, int rows, int nb, const double* D) {
  for (int r = threadIdx.x; r < rows; r += TF_THREADS) {
    double x[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) x[c] = (c < nb) ? ldg_cg(X + r + (size_t)c * ldx) : 0.0;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      if (c < nb) {
        x[c] = x[c] * D[NB + c * (NB + 1)];  // reciprocal of the diagonal (padding row)
#pragma unroll
        for (int c2 = c + 1; c2 < NB; ++c2)
          if (c2 < nb) x[c2] -= x[c] * D[c2 + c * (NB + 1)];
      }
    }
#pragma unroll
    for (int c = 0; c < NB; ++c)
      if (c < nb) X[r + (size_t)c * ldx] = x[c];
  }
}

// (the padding row NB of each column receives 1 / diagonal for row_solve: the row solves
// multiply by a reciprocal computed once per column instead of dividing in every row's
// dependency chain; exact whenever the diagonal is a power of two, as in the integer pins)
__device__ inline void load_lower_block(double* D, const double* A, int ld, int nb) {
  for (int e = threadIdx.x; e < NB * NB; e += TF_THREADS) {
    const int r = e % NB, c = e / NB;
    const double v = (r < nb && c < nb && r >= c) ? ldg_cg(A + r + (size_t)c * ld) : 0.0;
    D[r + c * (NB + 1)] = v;
    if (r == c) D[NB + c * (NB + 1)] = 1.0 / v;
  }
  __syncthreads();
}

// POTRF (DPOTF2): blocked left-looking Cholesky of the b x b tile A.
// Only the lower triangle is read or written (Z2).  Returns -1 or failing local column.
__device__ inline int potrf_left(const Ctx& cx, double* A, double* sm) {
  const int b = cx.b;
  double* D = sm + GemmNT32::SMEM_DOUBLES;  // (NB+1) x NB block after the engine buffers
  int* sflag = reinterpret_cast<int*>(D + (NB + 1) * NB);
  for (int jb = 0; jb < b; jb += NB) {
    const int nb = min(NB, b - jb);
    if (jb > 0) {
      for (int r0 = jb; r0 < b; r0 += 128) {
        GemmNT32 g;
        g.zero();
        const int mm = min(128, b - r0);
        g.run(sm, A + r0, b, A + jb, b, mm, nb, jb);
        sub_store(g, A + r0 + (size_t)jb * b, b, mm, nb, /*lower_mask=*/r0 < jb + nb, r0, jb);
      }
      __syncthreads();
    }
    load_lower_block(D, A + jb + (size_t)jb * b, b, nb);
    const int fail = chol_diag_block(D, nb, sflag);
    if (fail >= 0) return jb + fail;
    for (int e = threadIdx.x; e < nb * nb; e += TF_THREADS) {
      const int r = e % nb, c = e / nb;
      if (r >= c) A[jb + r + (size_t)(jb + c) * b] = D[r + c * (NB + 1)];
    }
    row_solve(A + jb + nb + (size_t)jb * b, b, b - jb - nb, nb, D);
    fence_proxy_async_all();  // the next column block's bulk copies read what was just stored
    __syncthreads();
  }
  return -1;
}

// POTRF for b a multiple of 128 (>= 256): right-looking over 128-column panels — each panel
// is factored left-looking in 32-column steps (K limited to the panel), then the trailing
// lower triangle takes the rank-128 update as 128x128 DMMA tiles (SYRK/GEMM shape, K = 128).
__device__ inline int potrf_right(const Ctx& cx, double* A, double* sm) {
  const int b = cx.b;
  double* D = sm + GemmNT32::SMEM_DOUBLES;
  int* sflag = reinterpret_cast<int*>(D + (NB + 1) * NB);
  for (int J = 0; J < b; J += 128) {
    for (int jb = J; jb < J + 128; jb += NB) {
      if (jb > J) {
        for (int r0 = jb; r0 < b; r0 += 128) {
          GemmNT32 g;
          g.zero();
          const int mm = min(128, b - r0);
          g.run(sm, A + r0 + (size_t)J * b, b, A + jb + (size_t)J * b, b, mm, NB, jb - J);
          sub_store(g, A + r0 + (size_t)jb * b, b, mm, NB, /*lower_mask=*/r0 < jb + NB, r0, jb);
        }
        __syncthreads();
      }
      load_lower_block(D, A + jb + (size_t)jb * b, b, NB);
      const int fail = chol_diag_block(D, NB, sflag);
      if (fail >= 0) return jb + fail;
      for (int e = threadIdx.x; e < NB * NB; e += TF_THREADS) {
        const int r = e % NB, c = e / NB;
        if (r >= c) A[jb + r + (size_t)(jb + c) * b] = D[r + c * (NB + 1)];
      }
      row_solve(A + jb + NB + (size_t)jb * b, b, b - jb - NB, NB, D);
      fence_proxy_async_all();
      __syncthreads();
    }
    // trailing lower triangle: C(mi, ni) -= L(mi, J:J+128) L(ni, J:J+128)^T
    for (int m0 = J + 128; m0 < b; m0 += 128)
      for (int n0 = J + 128; n0 <= m0; n0 += 128) {
        GemmNT128 g;
        g.zero();
        g.run(sm, A + m0 + (size_t)J * b, b, A + n0 + (size_t)J * b, b, 128, 128, 128);
        sub_store(g, A + m0 + (size_t)n0 * b, b, 128, 128, /*lower_mask=*/m0 == n0, m0, n0);
      }
    __syncthreads();
  }
  return -1;
}

// ---- b = 128 (config 1's tile size): POTRF and TRSM entirely in shared memory.  The tile
// is read once and written once; per 32-column block: warp 0's Cholesky of the diagonal
// block (chol_diag_block), row solves against it, and the rank-32 update of what remains
// by DMMA fragments read straight from shared memory (right-looking) — no global round
// trips and no operand pipeline start-up inside the tile.  Same operations per element as
// the blocked kernels above (products exact on the integer pins); rounding order differs.
constexpr int T128_LD = 132;  // column stride: the 32 lanes of a fragment load hit 16 banks twice

// row_solve on rows held in shared memory (X ld ldx), nb = NB
__device__ inline void row_solve_smem(double* X, int ldx, int rows, const double* D) {
  for (int r = threadIdx.x; r < rows; r += TF_THREADS) {
    double x[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) x[c] = X[r + c * ldx];
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      x[c] = x[c] * D[NB + c * (NB + 1)];
#pragma unroll
      for (int c2 = c + 1; c2 < NB; ++c2) x[c2] -= x[c] * D[c2 + c * (NB + 1)];
    }
#pragma unroll
    for (int c = 0; c < NB; ++c) X[r + c * ldx] = x[c];
  }
}

// C(8x8 fragment at rows r, columns cc of S, ld lds) -= sum_{k<32} A(r.., k) B(cc.., k), the
// A / B columns k at A + k * lda / B + k * ldb (one warp)
__device__ __forceinline__ void frag_rank32(double* S, int lds, int r, int cc, const double* Ak, int lda,
                                            const double* Bk, int ldb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  double c2[2] = {S[(r + g) + (size_t)(cc + 2 * q) * lds], S[(r + g) + (size_t)(cc + 2 * q + 1) * lds]};
  double a[8], bv[8];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    a[ks] = Ak[(r + g) + (size_t)(4 * ks + q) * lda];
    bv[ks] = Bk[(cc + g) + (size_t)(4 * ks + q) * ldb];
  }
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) dmma(c2, -a[ks], bv[ks]);
  S[(r + g) + (size_t)(cc + 2 * q) * lds] = c2[0];
  S[(r + g) + (size_t)(cc + 2 * q + 1) * lds] = c2[1];
}

__device__ inline int potrf_128(const Ctx& cx, double* A, double* sm, int lda = 128) {
  constexpr int LD = T128_LD;
  const int tid = threadIdx.x, warp = tid >> 5;
  double* T = sm;                          // 128 x LD
  double* D = T + 128 * LD;                // (NB+1) x NB
  int* sflag = reinterpret_cast<int*>(D + (NB + 1) * NB);
  TF_LU_T0();
  for (int e = tid; e < 128 * 64; e += TF_THREADS) {  // lower triangle (upper: zeros)
    const int r = (2 * e) % 128, c = (2 * e) / 128;
    const double2 v = __ldcg(reinterpret_cast<const double2*>(A + r + (size_t)c * lda));
    T[r + c * LD] = r >= c ? v.x : 0.0;
    T[r + 1 + c * LD] = r + 1 >= c ? v.y : 0.0;
  }
  __syncthreads();
  for (int jb = 0; jb < 128; jb += NB) {
    for (int e = tid; e < NB * NB; e += TF_THREADS) {
      const int r = e % NB, c = e / NB;
      D[r + c * (NB + 1)] = r >= c ? T[jb + r + (jb + c) * LD] : 0.0;
    }
    __syncthreads();
    TF_LU_T(0);
    const int fail = chol_diag_block(D, NB, sflag);
    TF_LU_T(1);
    if (fail >= 0) return jb + fail;
    for (int e = tid; e < NB * NB; e += TF_THREADS) {
      const int r = e % NB, c = e / NB;
      if (r >= c) T[jb + r + (jb + c) * LD] = D[r + c * (NB + 1)];
    }
    const int m0 = jb + NB, m = 128 - m0;
    if (m == 0) break;
    row_solve_smem(T + m0 + jb * LD, LD, m, D);
    __syncthreads();
    TF_LU_T(2);
    // trailing lower triangle (8x8 fragments on and below the block diagonal)
    const int nbk = m / 8, nfrag = nbk * (nbk + 1) / 2;
    for (int f = warp; f < nfrag; f += TF_WARPS) {
      int bi = (int)((sqrtf(8.0f * f + 1.0f) - 1.0f) * 0.5f);
      while ((bi + 1) * (bi + 2) / 2 <= f) ++bi;
      while (bi * (bi + 1) / 2 > f) --bi;
      const int bj = f - bi * (bi + 1) / 2;
      frag_rank32(T, LD, m0 + 8 * bi, m0 + 8 * bj, T + jb * LD, LD, T + jb * LD, LD);
    }
    __syncthreads();
    TF_LU_T(3);
  }
  __syncthreads();
  for (int e = tid; e < 128 * 128; e += TF_THREADS) {
    const int r = e % 128, c = e / 128;
    if (r >= c) A[r + (size_t)c * lda] = T[r + c * LD];
  }
  return -1;
}

// TRSM, b = 128: X (128 x 128) <- X L^{-T} in shared memory, right-looking over 32-column
// blocks: row solves of block jb against L's diagonal block, then X(:, jb+32:) -= X(:, jb
// block) L(jb+32:, jb block)^T by DMMA fragments from shared memory.
__device__ inline void trsm_128(const Ctx& cx, const double* L, double* X, double* sm, int ldl = 128, int ldx = 128) {
  constexpr int LD = T128_LD;
  const int tid = threadIdx.x, warp = tid >> 5;
  double* Xs = sm;                        // 128 x LD
  double* Ls = Xs + 128 * LD;             // L(jb.., jb block): 32 columns, ld LD
  double* D = Ls + NB * LD;               // (NB+1) x NB
  TF_LU_T0();
  for (int e = tid; e < 128 * 64; e += TF_THREADS) {
    const int r = (2 * e) % 128, c = (2 * e) / 128;
    const double2 v = __ldcg(reinterpret_cast<const double2*>(X + r + (size_t)c * ldx));
    Xs[r + c * LD] = v.x;
    Xs[r + 1 + c * LD] = v.y;
  }
  for (int jb = 0; jb < 128; jb += NB) {
    const int rows = 128 - jb;  // L rows jb .. 127 of the block's columns
    for (int e = tid; e < rows * NB; e += TF_THREADS) {
      const int r = e % rows, c = e / rows;
      Ls[r + c * LD] = ldg_cg(L + (jb + r) + (size_t)(jb + c) * ldl);
    }
    __syncthreads();
    for (int e = tid; e < NB * NB; e += TF_THREADS) {
      const int r = e % NB, c = e / NB;
      const double v = r >= c ? Ls[r + c * LD] : 0.0;
      D[r + c * (NB + 1)] = v;
      if (r == c) D[NB + c * (NB + 1)] = 1.0 / v;
    }
    __syncthreads();
    TF_LU_T(4);
    row_solve_smem(Xs + jb * LD, LD, 128, D);
    __syncthreads();
    TF_LU_T(5);
    const int n0 = jb + NB, ncol = 128 - n0;
    const int nfrag = 16 * (ncol / 8);
    for (int f = warp; f < nfrag; f += TF_WARPS) {
      const int bi = f % 16, bj = f / 16;
      frag_rank32(Xs, LD, 8 * bi, n0 + 8 * bj, Xs + jb * LD, LD, Ls - jb, LD);  // L(row, jb + k) = Ls[row - jb + k LD]
    }
    __syncthreads();
    TF_LU_T(6);
  }
  for (int e = tid; e < 128 * 64; e += TF_THREADS) {
    const int r = (2 * e) % 128, c = (2 * e) / 128;
    *reinterpret_cast<double2*>(X + r + (size_t)c * ldx) = make_double2(Xs[r + c * LD], Xs[r + 1 + c * LD]);
  }
  TF_LU_T(7);
}

// TRSM (DTRSM): rows [item*RB, +RB) of X <- X L^{-T}, left-looking over
// column blocks of NB: X[:,cb] -= X[:,<cb] L[cb,<cb]^T (DMMA), then the NB x NB solve.
__device__ inline void trsm_left(const Ctx& cx, const double* L, double* X, int item, double* sm) {
  const int b = cx.b;
  const int r0 = item * RB, rows = min(RB, b - r0);
  double* D = sm + GemmNT32::SMEM_DOUBLES;
  X += r0;
  for (int jb = 0; jb < b; jb += NB) {
    const int nb = min(NB, b - jb);
#ifdef TF_DEBUG_TRACE
    if (threadIdx.x == 0) printf("trsm blk %d jb %d\n", blockIdx.x, jb);
#endif
    if (jb > 0) {
      GemmNT32 g;
      g.zero();
      g.run(sm, X, b, L + jb, b, rows, nb, jb);
      sub_store(g, X + (size_t)jb * b, b, rows, nb);
    }
    load_lower_block(D, L + jb + (size_t)jb * b, b, nb);  // (has __syncthreads)
    row_solve(X + (size_t)jb * b, b, rows, nb, D);
    fence_proxy_async_all();  // the next block's bulk copies read the rows just solved
    __syncthreads();
  }
}

// the 128 x 128 shared-memory kernels on blocks of a larger tile, as separate variants (one
// register allocation each, like the other tile kernels)
TF_DEF_REF_RET(v_potrf_128ld, potrf_128, (Ctx cx, double* A, int lda), (cx, A, dsm, lda))
TF_DEF_REF(v_trsm_128ld, trsm_128, (Ctx cx, const double* L, double* X, int ldl, int ldx), (cx, L, X, dsm, ldl, ldx))

// POTRF for b a multiple of 128 (>= 256), left-looking over 128-column panels: the panel's
// rows take the update from all earlier panels as 128 x 128 DMMA-engine products with K = J
// (one long pipeline per row block), then its diagonal block is factored and the blocks
// below it solved entirely in shared memory (potrf_128, trsm_128).  Same operations per
// element as the right-looking form, in a different order (products exact on the pins).
__device__ inline int potrf_blocked(const Ctx& cx, double* A, double* sm) {
  const int b = cx.b;
  for (int J = 0; J < b; J += 128) {
    if (J > 0) {
      for (int r0 = J; r0 < b; r0 += 128) {
        GemmNT128 g;
        g.zero();
        g.run(sm, A + r0, b, A + J, b, 128, 128, J);
        sub_store(g, A + r0 + (size_t)J * b, b, 128, 128, /*lower_mask=*/r0 == J, r0, J);
      }
      __syncthreads();
    }
    const int f = potrf_128(cx, A + J + (size_t)J * b, sm, b);
    if (f >= 0) return J + f;
    fence_proxy_async_all();
    __syncthreads();
    for (int r0 = J + 128; r0 < b; r0 += 128) {
      v_trsm_128ld(cx, A + J + (size_t)J * b, A + r0 + (size_t)J * b, b, b);
      fence_proxy_async_all();
      __syncthreads();
    }
  }
  return -1;
}

// TRSM for b a multiple of 128 (>= 256): right-looking over 128-column panels as POTRF —
// each panel solved left-looking in 32-column steps (K limited to the panel), then the
// columns to its right take the rank-128 update as 128x128 DMMA tiles (K = 128).
__device__ inline void trsm_right(const Ctx& cx, const double* L, double* X, int item, double* sm) {
  const int b = cx.b;
  const int r0 = item * RB, rows = min(RB, b - r0);
  double* D = sm + GemmNT32::SMEM_DOUBLES;
  X += r0;
  if (rows == 128) {
    // left-looking over 128-column panels: X(:, J:J+128) -= X(:, 0:J) L(J:J+128, 0:J)^T as ONE
    // DMMA-engine product with K = J (fewer, longer pipelines than a rank-128 update per panel
    // pair), then the panel's 128 x 128 block solved entirely in shared memory (trsm_128)
    for (int J = 0; J < b; J += 128) {
      if (J > 0) {
        GemmNT128 g;
        g.zero();
        g.run(sm, X, b, L + J, b, rows, 128, J);
        sub_store(g, X + (size_t)J * b, b, rows, 128);
        __syncthreads();
      }
      v_trsm_128ld(cx, L + J + (size_t)J * b, X + (size_t)J * b, b, b);
      fence_proxy_async_all();
      __syncthreads();
    }
    return;
  }
  for (int J = 0; J < b; J += 128) {
    {
      for (int jb = J; jb < J + 128; jb += NB) {
        if (jb > J) {
          GemmNT32 g;
          g.zero();
          g.run(sm, X + (size_t)J * b, b, L + jb + (size_t)J * b, b, rows, NB, jb - J);
          sub_store(g, X + (size_t)jb * b, b, rows, NB);
        }
        load_lower_block(D, L + jb + (size_t)jb * b, b, NB);  // (has __syncthreads)
        row_solve(X + (size_t)jb * b, b, rows, NB, D);
        fence_proxy_async_all();
        __syncthreads();
      }
    }
    // columns to the right: X(:, n0:n0+128) -= X(:, J:J+128) L(n0:n0+128, J:J+128)^T
    for (int n0 = J + 128; n0 < b; n0 += 128) {
      GemmNT128 g;
      g.zero();
      g.run(sm, X + (size_t)J * b, b, L + n0 + (size_t)J * b, b, rows, 128, 128);
      sub_store(g, X + (size_t)n0 * b, b, rows, 128);
    }
    __syncthreads();
  }
}

// Panel-level Cholesky DAG (tf_sched.h K_POTRF_D / K_POTRF_B / K_TRSM_P): the bodies of
// potrf_blocked's and trsm_right's panel loops as separate work items, so every element sees
// the same operations in the same order as in the one-item kernels (bitwise identical).
// Diagonal block of panel Jp: update from the panels to its left (K = J), then potrf_128.
__device__ inline int potrf_panel_diag(const Ctx& cx, double* A, int Jp, double* sm) {
  const int b = cx.b, J = Jp * 128;
  if (J > 0) {
    GemmNT128 g;
    g.zero();
    g.run(sm, A + J, b, A + J, b, 128, 128, J);
    sub_store(g, A + J + (size_t)J * b, b, 128, 128, /*lower_mask=*/true, J, J);
    __syncthreads();
  }
  const int f = potrf_128(cx, A + J + (size_t)J * b, sm, b);
  fence_proxy_async_all();
  __syncthreads();
  return f >= 0 ? J + f : -1;
}
// Block row r0 = J + 128 (item + 1) of panel Jp: the same update, then the solve against the
// factored diagonal block.
__device__ inline void potrf_panel_below(const Ctx& cx, double* A, int Jp, int item, double* sm) {
  const int b = cx.b, J = Jp * 128, r0 = J + 128 * (item + 1);
  if (J > 0) {
    GemmNT128 g;
    g.zero();
    g.run(sm, A + r0, b, A + J, b, 128, 128, J);
    sub_store(g, A + r0 + (size_t)J * b, b, 128, 128, /*lower_mask=*/false, r0, J);
    __syncthreads();
  }
  v_trsm_128ld(cx, A + J + (size_t)J * b, A + r0 + (size_t)J * b, b, b);
  fence_proxy_async_all();
  __syncthreads();
}
// Panel Jp of TRSM row block `item` (trsm_right's full-row-block loop body).
__device__ inline void trsm_panel(const Ctx& cx, const double* L, double* X, int Jp, int item, double* sm) {
  const int b = cx.b, J = Jp * 128;
  X += item * RB;
  if (J > 0) {
    GemmNT128 g;
    g.zero();
    g.run(sm, X, b, L + J, b, 128, 128, J);
    sub_store(g, X + (size_t)J * b, b, 128, 128);
    __syncthreads();
  }
  v_trsm_128ld(cx, L + J + (size_t)J * b, X + (size_t)J * b, b, b);
  fence_proxy_async_all();
  __syncthreads();
}
TF_DEF_REF_RET(v_potrf_pd, potrf_panel_diag, (Ctx cx, double* A, int Jp), (cx, A, Jp, dsm))
TF_DEF_REF(v_potrf_pb, potrf_panel_below, (Ctx cx, double* A, int Jp, int item), (cx, A, Jp, item, dsm))
TF_DEF_REF(v_trsm_p, trsm_panel, (Ctx cx, const double* L, double* X, int Jp, int item), (cx, L, X, Jp, item, dsm))

// SYRK (DGSMM with i = j): lower sub-tile `item` of C -= A A^T.
__device__ inline void syrk_body(const Ctx& cx, const double* A, double* C, int item, double* sm) {
  const int b = cx.b;
  int mi = 0, rem = item;
  while (rem > mi) { rem -= mi + 1; ++mi; }
  const int ni = rem;  // mi >= ni
  const int m0 = mi * RB, n0 = ni * RB;
  const int mm = min(RB, b - m0), nn = min(RB, b - n0);
  prefetch_l2(C + m0 + (size_t)n0 * b, b, mm, nn);
  GemmNT128 g;
  g.zero();
  g.run(sm, A + m0, b, A + n0, b, mm, nn, b);
  sub_store(g, C + m0 + (size_t)n0 * b, b, mm, nn, /*lower_mask=*/mi == ni, m0, n0, /*red=*/true);
}

// GEMM (DGSMM with i > j): sub-tile `item` of C -= A B^T.
__device__ inline void gemm_body(const Ctx& cx, const double* A, const double* B, double* C, int item,
                                 double* sm) {
  const int b = cx.b;
  const int nr = ceil_div(b, RB);
  const int gs = gemm_group(b);
  if (gs > 1) {
    // gs 128x128 sub-tiles (same rows, adjacent columns) per item, run as one continuous
    // slice stream (Gemm::chain): each warp's epilogue of sub-tile x overlaps the other
    // warps' DMMAs, and the scheduler round trip is paid once per group
    const int mi = item % nr, nj = item / nr;
    const int m0 = mi * RB, mm = min(RB, b - m0);
    for (int x = 0; x < gs; ++x) {
      const int n = (nj * gs + x) * RB;
      prefetch_l2(C + m0 + (size_t)n * b, b, mm, min(RB, b - n));
    }
    const int n0 = nj * gs * RB;
    GemmNT128 g;
    g.chain(sm, A + m0, b, B + n0, b, gs, mm, min(gs * RB, b - n0), b, [&](int x) {
      if (x >= 0) {
#ifndef TF_KB_NOEPI
        const int n = n0 + x * RB;
        sub_store(g, C + m0 + (size_t)n * b, b, mm, min(RB, b - n), false, 0, 0, /*red=*/true);
#else
        double s = 0.0;  // kbench probe only: keep the products live without an epilogue
        g.for_each(mm, RB, [&](int, int, double v) { s += v; });
        if (s == 1234.5) C[threadIdx.x] = s;
#endif
      }
      g.zero();
    });
    return;
  }
  const int mi = item % nr, ni = item / nr;
  const int m0 = mi * RB, n0 = ni * RB;
  const int mm = min(RB, b - m0), nn = min(RB, b - n0);
#ifdef TF_PROBE
  unsigned long long t0 = probe_now();
#endif
  prefetch_l2(C + m0 + (size_t)n0 * b, b, mm, nn);
  GemmNT128 g;
  g.zero();
  TF_PROBE_MARK(0, t0);
  g.run(sm, A + m0, b, B + n0, b, mm, nn, b);
  TF_PROBE_MARK(1, t0);
  sub_store(g, C + m0 + (size_t)n0 * b, b, mm, nn, false, 0, 0, /*red=*/true);
  __syncthreads();
  TF_PROBE_MARK(2, t0);
}

// GEMM, the whole tile C -= A B^T as one work item (b a multiple of 128, operands 16-byte
// aligned): the nr x nr sub-tile products of gemm_body run as one continuous slice stream
// (Gemm::chain2_mb), row strip by row strip.  Same arithmetic per sub-tile as gemm_body.
// Used by the panel-level Cholesky graph for the updates of steps with enough tiles to keep
// every SM busy with whole-tile items (tf_host.cpp).
__device__ inline void gemm_tile_body(const Ctx& cx, const double* A, const double* B, double* C, double* sm) {
  const int b = cx.b;
  const int nr = b / RB;
  GemmNT128 g;
  g.chain2_mb<2>(sm, A, b, B, b, nr * nr, nr, b, [&](int x) {
    // the C strip of the products about to start: into L2 ahead of their epilogues
    if (x < 0 || (x + 1) % nr == 0) {
      const int mi = (x + 1) / nr;
      if (mi < nr)
        for (int nj = 0; nj < nr; ++nj) prefetch_l2(C + mi * RB + (size_t)(nj * RB) * b, b, RB, RB);
    }
    if (x >= 0) {
      const int mi = x / nr, nj = x - mi * nr;
      sub_store(g, C + mi * RB + (size_t)(nj * RB) * b, b, RB, RB, false, 0, 0, /*red=*/true);
    }
    g.zero();
  });
}

TF_DEF_REF_RET(v_potrf_left, potrf_left, (Ctx cx, double* A), (cx, A, dsm))
TF_DEF_REF_RET(v_potrf_right, potrf_right, (Ctx cx, double* A), (cx, A, dsm))
TF_DEF_REF(v_trsm_left, trsm_left, (Ctx cx, const double* L, double* X, int item), (cx, L, X, item, dsm))
TF_DEF_REF(v_trsm_right, trsm_right, (Ctx cx, const double* L, double* X, int item), (cx, L, X, item, dsm))
TF_DEF_REF_RET(v_potrf_128, potrf_128, (Ctx cx, double* A), (cx, A, dsm))
TF_DEF_REF_RET(v_potrf_blocked, potrf_blocked, (Ctx cx, double* A), (cx, A, dsm))
TF_DEF_REF(v_trsm_128, trsm_128, (Ctx cx, const double* L, double* X), (cx, L, X, dsm))
TF_DEF_REF(v_syrk, syrk_body, (Ctx cx, const double* A, double* C, int item), (cx, A, C, item, dsm))
TF_DEF_REF(v_gemm, gemm_body, (Ctx cx, const double* A, const double* B, double* C, int item), (cx, A, B, C, item, dsm))
TF_DEF_REF(v_gemm_tile, gemm_tile_body, (Ctx cx, const double* A, const double* B, double* C), (cx, A, B, C, dsm))

// Cholesky task kernels (the `sm` argument is the caller's dynamic shared memory; the
// variants re-declare it).  POTRF / TRSM: right-looking over 128-column panels for b a
// multiple of 128 (>= 256), left-looking 32-column blocks otherwise.
__device__ inline int potrf_item(const Ctx& cx, double* A, double*) {
  if (cx.b == 128) return v_potrf_128(cx, A);
  if (cx.b < 256 || cx.b % 128) return v_potrf_left(cx, A);
#ifdef TF_POTRF_RIGHT
  return v_potrf_right(cx, A);
#else
  return v_potrf_blocked(cx, A);
#endif
}
__device__ inline void trsm_item(const Ctx& cx, const double* L, double* X, int item, double*) {
  if (cx.b == 128) v_trsm_128(cx, L, X);
  else if (cx.b < 256 || cx.b % 128) v_trsm_left(cx, L, X, item);
  else v_trsm_right(cx, L, X, item);
}
__device__ inline void syrk_item(const Ctx& cx, const double* A, double* C, int item, double*) { v_syrk(cx, A, C, item); }
__device__ inline void gemm_item(const Ctx& cx, const double* A, const double* B, double* C, int item, double*) {
  v_gemm(cx, A, B, C, item);
}

// ====================================================================================
// QR (C2)
// ====================================================================================

// Householder scalars (dlarfg without safmin rescaling).
struct House {
  double tau, beta, den;
};
__device__ __forceinline__ House make_house(double alpha, double ss) {
  House h;
  if (ss == 0.0) { h.tau = 0.0; h.beta = alpha; h.den = 1.0; return h; }
  const double xn = sqrt(ss);
  const double nrm = sqrt(alpha * alpha + xn * xn);
  h.beta = (alpha >= 0.0) ? -nrm : nrm;
  h.tau = (h.beta - alpha) / h.beta;
  h.den = alpha - h.beta;
  return h;
}

// Panel of DGEQRT: P is the (mp x ib) panel A[c0:b, c0:c1] (ld ldp,
// shared or global), Ts the ib x ib T block (smem, ld ib, pre-zeroed).
__device__ inline void geqrt_panel(double* P, int ldp, int mp, int ib, double* Ts, double* red, double* sdot) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int jj = 0; jj < ib; ++jj) {
    double ss = 0.0;
    for (int r = jj + 1 + tid; r < mp; r += TF_THREADS) {
      const double x = P[r + (size_t)jj * ldp];
      ss += x * x;
    }
    ss = block_sum(ss, red);
    const double alpha = P[jj + (size_t)jj * ldp];
    const House h = make_house(alpha, ss);
    __syncthreads();
    if (ss != 0.0) {
      for (int r = jj + 1 + tid; r < mp; r += TF_THREADS) P[r + (size_t)jj * ldp] = P[r + (size_t)jj * ldp] / h.den;
      if (tid == 0) P[jj + (size_t)jj * ldp] = h.beta;
    }
    __syncthreads();
    for (int c = warp; c < ib; c += TF_WARPS) {
      if (c == jj) continue;
      double s = 0.0;
      for (int r = jj + 1 + lane; r < mp; r += 32) s += P[r + (size_t)jj * ldp] * P[r + (size_t)c * ldp];
      s = warp_sum(s);
      if (lane == 0) sdot[c] = P[jj + (size_t)c * ldp] + s;
    }
    __syncthreads();
    const int nr = mp - jj, ncol = ib - jj - 1;
    for (int e = tid; e < nr * ncol; e += TF_THREADS) {
      const int r = jj + e % nr, c = jj + 1 + e / nr;
      const double tw = h.tau * sdot[c];
      if (r == jj) P[jj + (size_t)c * ldp] -= tw;
      else P[r + (size_t)c * ldp] -= tw * P[r + (size_t)jj * ldp];
    }
    if (tid < jj) {
      double s = 0.0;
      for (int m = tid; m < jj; ++m) s += Ts[tid + m * ib] * (-h.tau * sdot[m]);
      Ts[tid + jj * ib] = s;
    }
    if (tid == 0) Ts[jj + jj * ib] = h.tau;
    __syncthreads();
  }
}

// GEQRT with inner block ib.  Writes the explicit unit-lower copy of
// V (VX, b x b) for the LARFB items of this step.
__device__ inline void geqrt_ref(const Ctx& cx, double* A, double* Tst, double* VX, double* sm) {
  const int b = cx.b, ib = cx.ib, tid = threadIdx.x;
  double* W = cx.scratch;
  double* W2 = W + (size_t)ib * b;
  for (int c0 = 0; c0 < b; c0 += ib) {
    const int c1 = c0 + ib, mp = b - c0;
    const bool in_smem = (size_t)mp * ib + (size_t)ib * ib + 2 * TF_WARPS + ib <= SMEM_USER;
    double* Ts = sm;
    double* red = Ts + ib * ib;
    double* sdot = red + TF_WARPS;
    double* P = sdot + ib + TF_WARPS;
    int ldp = mp;
    for (int e = tid; e < ib * ib; e += TF_THREADS) Ts[e] = 0.0;
    if (in_smem) {
      for (int e = tid; e < mp * ib; e += TF_THREADS) {
        const int r = e % mp, c = e / mp;
        P[e] = ldg_cg(A + c0 + r + (size_t)(c0 + c) * b);
      }
    } else {
      P = A + c0 + (size_t)c0 * b;
      ldp = b;
    }
    __syncthreads();
    geqrt_panel(P, ldp, mp, ib, Ts, red, sdot);
    if (in_smem) {
      for (int e = tid; e < mp * ib; e += TF_THREADS) {
        const int r = e % mp, c = e / mp;
        A[c0 + r + (size_t)(c0 + c) * b] = P[e];
      }
    }
    for (int e = tid; e < ib * ib; e += TF_THREADS) Tst[(size_t)c0 * ib + e] = Ts[e];
    for (int e = tid; e < mp * ib; e += TF_THREADS) {
      const int r = e % mp, m = e / mp;  // tile row c0 + r, column c0 + m
      const double v = (r < m) ? 0.0 : (r == m ? 1.0 : P[r + (size_t)m * ldp]);
      VX[c0 + r + (size_t)(c0 + m) * b] = v;
    }
    __syncthreads();
    if (c1 < b) {
      // W = V_s^T A[c0:b, c1:b];  W2 = T_s^T W;  A[c0:b, c1:b] -= V_s W2
      w_product(sm, W, ib, VX + c0 + (size_t)c0 * b, b, A + c0 + (size_t)c1 * b, b, ib, b - c1, mp, nullptr, 0);
      double* sT = sm;
      load_ts(sT, Tst, ib, c0);
      apply_tt(sT, ib, W, W2, ib, b - c1);
      update_mn(sm, A + c0 + (size_t)c1 * b, b, VX + c0 + (size_t)c0 * b, b, W2, ib, mp, b - c1, ib);
      __syncthreads();
    }
  }
}

// LARFB: slab `item` of C <- Q_kk^T C, s = 0..t-1 (reading Z5).
__device__ inline void larfb_ref(const Ctx& cx, const double* VX, const double* Tst, double* C, int item,
                                  double* sm) {
  const int b = cx.b, ib = cx.ib;
  const int n0 = item * NS, nc = min(NS, b - n0);
  double* W = cx.scratch;
  double* W2 = W + (size_t)ib * b;
  C += (size_t)n0 * b;
  for (int c0 = 0; c0 < b; c0 += ib) {
    const int mp = b - c0;
    w_product(sm, W, ib, VX + c0 + (size_t)c0 * b, b, C + c0, b, ib, nc, mp, nullptr, 0);
    load_ts(sm, Tst, ib, c0);
    apply_tt(sm, ib, W, W2, ib, nc);
    update_mn(sm, C + c0, b, VX + c0 + (size_t)c0 * b, b, W2, ib, mp, nc, ib);
    __syncthreads();
  }
}

// Panel of DTSQRT: bottom P (b x ib, ld ldp), top Rb (ib x ib, ld ib,
// upper triangle = R[c0:c1, c0:c1]), T block Ts (ld ib, pre-zeroed).
__device__ inline void tsqrt_panel(double* P, int ldp, int b, double* Rb, int ib, double* Ts, double* red,
                                   double* sdot) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef TF_PROBE
  unsigned long long t0 = probe_now();
#endif
  for (int jj = 0; jj < ib; ++jj) {
    double ss = 0.0;
    for (int r = tid; r < b; r += TF_THREADS) {
      const double x = P[r + (size_t)jj * ldp];
      ss += x * x;
    }
    ss = block_sum(ss, red);
    TF_PROBE_MARK(4, t0);
    const double alpha = Rb[jj + jj * ib];
    const House h = make_house(alpha, ss);
    __syncthreads();
    TF_PROBE_MARK(5, t0);
    if (ss != 0.0) {
      for (int r = tid; r < b; r += TF_THREADS) P[r + (size_t)jj * ldp] = P[r + (size_t)jj * ldp] / h.den;
      if (tid == 0) Rb[jj + jj * ib] = h.beta;
    }
    __syncthreads();
    for (int c = warp; c < ib; c += TF_WARPS) {
      if (c == jj) continue;
      double s = 0.0;
      for (int r = lane; r < b; r += 32) s += P[r + (size_t)jj * ldp] * P[r + (size_t)c * ldp];
      s = warp_sum(s);
      if (lane == 0) sdot[c] = (c > jj) ? Rb[jj + c * ib] + s : s;
    }
    __syncthreads();
    TF_PROBE_MARK(6, t0);
    const int ncol = ib - jj - 1;
    for (int e = tid; e < b * ncol; e += TF_THREADS) {
      const int r = e % b, c = jj + 1 + e / b;
      P[r + (size_t)c * ldp] -= (h.tau * sdot[c]) * P[r + (size_t)jj * ldp];
    }
    for (int c = jj + 1 + tid; c < ib; c += TF_THREADS) Rb[jj + c * ib] -= h.tau * sdot[c];
    if (tid < jj) {
      double s = 0.0;
      for (int m = tid; m < jj; ++m) s += Ts[tid + m * ib] * (-h.tau * sdot[m]);
      Ts[tid + jj * ib] = s;
    }
    if (tid == 0) Ts[jj + jj * ib] = h.tau;
    __syncthreads();
    TF_PROBE_MARK(7, t0);
  }
}

// TSQRT (inner blocking PAPER.md:637-647): QR of [R; A].  Reads and
// writes only the upper region of the diagonal tile R.
__device__ inline void tsqrt_ref(const Ctx& cx, double* R, double* A, double* Tst, double* sm) {
  const int b = cx.b, ib = cx.ib, tid = threadIdx.x;
  double* W = cx.scratch;
  double* W2 = W + (size_t)ib * b;
#ifdef TF_PROBE
  unsigned long long t0 = probe_now();
#endif
  for (int c0 = 0; c0 < b; c0 += ib) {
    const int c1 = c0 + ib;
    double* Ts = sm;
    double* Rb = Ts + ib * ib;
    double* red = Rb + ib * ib;
    double* sdot = red + TF_WARPS;
    double* P = sdot + ib + TF_WARPS;
    const bool in_smem = (size_t)b * ib + 2 * (size_t)ib * ib + 2 * TF_WARPS + ib <= SMEM_USER;
    int ldp = b;
    for (int e = tid; e < ib * ib; e += TF_THREADS) {
      const int r = e % ib, c = e / ib;
      Ts[e] = 0.0;
      Rb[e] = (r <= c) ? ldg_cg(R + c0 + r + (size_t)(c0 + c) * b) : 0.0;
    }
    if (in_smem) {
      for (int e = tid; e < b * ib; e += TF_THREADS) P[e] = ldg_cg(A + (size_t)c0 * b + e);
    } else {
      P = A + (size_t)c0 * b;
    }
    __syncthreads();
    TF_PROBE_MARK(3, t0);
    tsqrt_panel(P, ldp, b, Rb, ib, Ts, red, sdot);
    TF_PROBE_MARK(0, t0);
    if (in_smem)
      for (int e = tid; e < b * ib; e += TF_THREADS) A[(size_t)c0 * b + e] = P[e];
    for (int e = tid; e < ib * ib; e += TF_THREADS) {
      const int r = e % ib, c = e / ib;
      if (r <= c) R[c0 + r + (size_t)(c0 + c) * b] = Rb[e];
      Tst[(size_t)c0 * ib + e] = Ts[e];
    }
    __syncthreads();
    if (c1 < b) {
      // W = R[c0:c1, c1:b] + V_s^T A[:, c1:b]; W2 = T_s^T W; R -= W2; A[:, c1:b] -= V_s W2
      w_product(sm, W, ib, A + (size_t)c0 * b, b, A + (size_t)c1 * b, b, ib, b - c1, b, R + c0 + (size_t)c1 * b, b);
      TF_PROBE_MARK(1, t0);
      load_ts(sm, Tst, ib, c0);
      apply_tt(sm, ib, W, W2, ib, b - c1);
      for (int e = tid; e < ib * (b - c1); e += TF_THREADS) {
        const int m = e % ib, n = e / ib;
        double* p = R + c0 + m + (size_t)(c1 + n) * b;
        *p = ldg_cg(p) - W2[e];
      }
      update_mn(sm, A + (size_t)c1 * b, b, A + (size_t)c0 * b, b, W2, ib, b, b - c1, ib);
      __syncthreads();
      TF_PROBE_MARK(2, t0);
    }
  }
}

// SSRFB reference-blocked path: slab `item` of
// [R; A] <- Q_ik^T [R; A] (tile sizes the register-slab kernels do not cover).
__device__ inline void ssrfb_ref(const Ctx& cx, const double* V, const double* Tst, double* R, double* A,
                                 int item, double* sm) {
  const int b = cx.b, ib = cx.ib, tid = threadIdx.x;
  const int n0 = item * NS, nc = min(NS, b - n0);
  double* W = cx.scratch;
  double* W2 = W + (size_t)ib * b;
  R += (size_t)n0 * b;
  A += (size_t)n0 * b;
  for (int c0 = 0; c0 < b; c0 += ib) {
    w_product(sm, W, ib, V + (size_t)c0 * b, b, A, b, ib, nc, b, R + c0, b);
    load_ts(sm, Tst, ib, c0);
    apply_tt(sm, ib, W, W2, ib, nc);
    for (int e = tid; e < ib * nc; e += TF_THREADS) {
      const int m = e % ib, n = e / ib;
      double* p = R + c0 + m + (size_t)n * b;
      *p = ldg_cg(p) - W2[e];
    }
    update_mn(sm, A, b, V + (size_t)c0 * b, b, W2, ib, b, nc, ib);
    __syncthreads();
  }
}

}  // namespace tf
#include "tf_qr_slab.cuh"
namespace tf {

// QR task kernels: the register-slab path for b in {128, 256, 512} and ib in {32, 64}
// (ssrfb_reg_ok), the reference-blocked kernels otherwise.
#define TF_SLAB_DISPATCH(fn, ...)                      \
  do {                                                 \
    if (cx.b == 512) fn<4>(__VA_ARGS__);               \
    else if (cx.b == 256) fn<2>(__VA_ARGS__);          \
    else fn<1>(__VA_ARGS__);                           \
  } while (0)

TF_DEF_VARIANT(v_qr_slab, qr_slab,
               (Ctx cx, bool ts, double* A, double* R, double* Tst, double* VX, int cb, int ce),
               (cx, ts, A, R, Tst, VX, cb, ce, dsm))
TF_DEF_VARIANT(v_larfb_reg, larfb_reg, (Ctx cx, const double* VX, const double* Tst, double* C, int item),
               (cx, VX, Tst, C, item, dsm))
TF_DEF_VARIANT(v_ssrfb_reg, ssrfb_reg, (Ctx cx, const double* V, const double* Tst, double* R, double* A, int item),
               (cx, V, Tst, R, A, item, dsm))
TF_DEF_VARIANT(v_ssrfb_mirror, ssrfb_mirror,
               (Ctx cx, const double* V, const double* Tst, double* R, double* A, int item), (cx, V, Tst, R, A, item, dsm))
TF_DEF_REF(v_geqrt_ref, geqrt_ref, (Ctx cx, double* A, double* Tst, double* VX), (cx, A, Tst, VX, dsm))
TF_DEF_REF(v_larfb_ref, larfb_ref, (Ctx cx, const double* VX, const double* Tst, double* C, int item),
           (cx, VX, Tst, C, item, dsm))
TF_DEF_REF(v_tsqrt_ref, tsqrt_ref, (Ctx cx, double* R, double* A, double* Tst), (cx, R, A, Tst, dsm))
TF_DEF_REF(v_ssrfb_ref, ssrfb_ref, (Ctx cx, const double* V, const double* Tst, double* R, double* A, int item),
           (cx, V, Tst, R, A, item, dsm))

// GEQRT: A_kk -> V_kk, R_kk, T_kk; writes the unit-lower V copy VX.
__device__ inline void geqrt_item(const Ctx& cx, double* A, double* Tst, double* VX, double* sm) {
  if (ssrfb_reg_ok(cx.b, cx.ib)) TF_SLAB_DISPATCH(v_qr_slab, cx, false, A, nullptr, Tst, VX, 0, cx.b);
  else v_geqrt_ref(cx, A, Tst, VX);
}
// GEQRT slab task of the slab-level DAG: 32-column slab s (register-slab path only).
__device__ inline void geqrt_slab_item(const Ctx& cx, double* A, double* Tst, double* VX, int s, double* sm) {
  TF_SLAB_DISPATCH(v_qr_slab, cx, false, A, nullptr, Tst, VX, s * NSR, (s + 1) * NSR);
}
// LARFB: slab `item` of C <- Q_kk^T C.
__device__ inline void larfb_item(const Ctx& cx, const double* VX, const double* Tst, double* C, int item,
                                  double* sm) {
  if (ssrfb_reg_ok(cx.b, cx.ib)) TF_SLAB_DISPATCH(v_larfb_reg, cx, VX, Tst, C, item);
  else v_larfb_ref(cx, VX, Tst, C, item);
}
// TSQRT: QR of [R_kk; A_ik]; only the upper region of R_kk is touched.
__device__ inline void tsqrt_item(const Ctx& cx, double* R, double* A, double* Tst, double* sm) {
  if (ssrfb_reg_ok(cx.b, cx.ib)) TF_SLAB_DISPATCH(v_qr_slab, cx, true, A, R, Tst, nullptr, 0, cx.b);
  else v_tsqrt_ref(cx, R, A, Tst);
}
// Slab-level DAG, TSQRT slab s of [R_kk; A_ik].
__device__ inline void tsqrt_slab_item(const Ctx& cx, double* R, double* A, double* Tst, int s, double* sm) {
  TF_SLAB_DISPATCH(v_qr_slab, cx, true, A, R, Tst, nullptr, s * NSR, (s + 1) * NSR);
}
// SSRFB: slab `item` of [R_kj; A_ij] <- Q_ik^T [R_kj; A_ij].
__device__ inline void ssrfb_item(const Ctx& cx, const double* V, const double* Tst, double* R, double* A,
                                  int item, double* sm) {
#ifdef TF_SSRFB_SLAB
  if (ssrfb_reg_ok(cx.b, cx.ib)) TF_SLAB_DISPATCH(v_ssrfb_reg, cx, V, Tst, R, A, item);
#else
  if (ssrfb_reg_ok(cx.b, cx.ib)) TF_SLAB_DISPATCH(v_ssrfb_mirror, cx, V, Tst, R, A, item);
#endif
  else v_ssrfb_ref(cx, V, Tst, R, A, item);
}

// ====================================================================================
// LU (C3)
// ====================================================================================

// Rows c0..c0+ib of U (ld ldu) and the touched rows of A (ld lda) over columns [0, ncol):
// apply the pairwise swaps of block (jslot[jj] >= 0: top row jj <-> A row srow[jslot]),
// then U_s <- (I + Lb)^{-1} U_s with Lb strictly lower (smem, ld ib).  Staged through
// shared memory in column chunks; the unit-lower solve is right-looking with the rows
// of a column split over G lanes of one warp, subtraction order m = 0..r-1 as in C3.
__device__ inline void swap_solve(double* U, int ldu, double* A, int lda, int ib, int ncol, const int* jslot,
                                  const int* srow, int nslot, const double* Lb, double* buf, int bufcap) {
  const int tid = threadIdx.x;
  int cw = TF_THREADS;
  while (cw > 16 && (ib + nslot) * cw > bufcap) cw >>= 1;
  const int G = TF_THREADS / cw;  // lanes per column (power of two, <= 32)
  double* sU = buf;
  double* sA = buf + ib * cw;
  for (int cs = 0; cs < ncol; cs += cw) {
    const int w = min(cw, ncol - cs);
    for (int e = tid; e < ib * w; e += TF_THREADS) {
      const int m = e % ib, c = e / ib;
      sU[m + c * ib] = ldg_cg(U + m + (size_t)(cs + c) * ldu);
    }
    for (int e = tid; e < nslot * w; e += TF_THREADS) {
      const int s = e % nslot, c = e / nslot;
      sA[s + c * nslot] = ldg_cg(A + srow[s] + (size_t)(cs + c) * lda);
    }
    __syncthreads();
    const int c = tid / G, g = tid % G;
    const bool act = c < w;
    if (act && g == 0 && jslot) {
      for (int jj = 0; jj < ib; ++jj)
        if (jslot[jj] >= 0) {
          double t = sU[jj + c * ib];
          sU[jj + c * ib] = sA[jslot[jj] + c * nslot];
          sA[jslot[jj] + c * nslot] = t;
        }
    }
    for (int m = 0; m < ib; ++m) {
      __syncwarp();  // the G lanes of a column are consecutive lanes of one warp
      if (act) {
        const double xm = sU[m + c * ib];
        for (int r = m + 1 + g; r < ib; r += G) sU[r + c * ib] -= Lb[r + m * ib] * xm;
      }
    }
    __syncthreads();
    for (int e = tid; e < ib * w; e += TF_THREADS) {
      const int m = e % ib, cc = e / ib;
      U[m + (size_t)(cs + cc) * ldu] = sU[e];
    }
    for (int e = tid; e < nslot * w; e += TF_THREADS) {
      const int s = e % nslot, cc = e / nslot;
      A[srow[s] + (size_t)(cs + cc) * lda] = sA[e];
    }
    __syncthreads();
  }
}

// Build the swap slots of inner block [c0, c0+ib) from TSTRF pivots (values > b name
// bottom row ipiv-b-1).  rowslot: smem int[b] scratch.  Returns nslot.
__device__ inline int build_slots(const int* ipiv, int c0, int ib, int b, int* jslot, int* srow, int* rowslot,
                                  int* snslot) {
  for (int r = threadIdx.x; r < b; r += TF_THREADS) rowslot[r] = -1;
  __syncthreads();
  if (threadIdx.x == 0) {
    int ns = 0;
    for (int jj = 0; jj < ib; ++jj) {
      const int pv = ipiv[c0 + jj];
      if (pv > b) {
        const int r = pv - b - 1;
        if (rowslot[r] < 0) { rowslot[r] = ns; srow[ns++] = r; }
        jslot[jj] = rowslot[r];
      } else {
        jslot[jj] = -1;
      }
    }
    *snslot = ns;
  }
  __syncthreads();
  return *snslot;
}

// GETRF: LAPACK dgetrf semantics with block ib, whole-tile-row swaps
// (Z12), first-max pivot (Z11).  Writes LX (explicit unit-lower copy of L_kk) for the
// GESSM items.  Returns the first zero-pivot local column or -1.
__device__ inline int getrf_ref(const Ctx& cx, double* A, int* ipiv, double* LX, double* sm) {
  const int b = cx.b, ib = cx.ib, tid = threadIdx.x;
  double* redv = sm;
  int* redi = reinterpret_cast<int*>(redv + TF_WARPS);
  int first_zero = -1;
  for (int c0 = 0; c0 < b; c0 += ib) {
    const int c1 = c0 + ib;
    for (int j = c0; j < c1; ++j) {
      double v = -1.0;
      int idx = INT_MAX;
      for (int r = j + tid; r < (cx.nopiv ? j + 1 : b); r += TF_THREADS) amax_merge(v, idx, fabs(A[r + (size_t)j * b]), r);
      const int pr = block_amax(v, idx, redv, redi);
      const double pv = A[pr + (size_t)j * b];
      __syncthreads();
      if (tid == 0) ipiv[j] = pr + 1;
      if (pv != 0.0) {
        if (pr != j)
          for (int c = tid; c < b; c += TF_THREADS) {
            const double t = A[j + (size_t)c * b];
            A[j + (size_t)c * b] = A[pr + (size_t)c * b];
            A[pr + (size_t)c * b] = t;
          }
        __syncthreads();
        const double ajj = A[j + (size_t)j * b];
        for (int r = j + 1 + tid; r < b; r += TF_THREADS) A[r + (size_t)j * b] = A[r + (size_t)j * b] / ajj;
      } else if (first_zero < 0) {
        first_zero = j;
      }
      __syncthreads();
      const int nr = b - j - 1, ncol = c1 - j - 1;
      for (int e = tid; e < nr * ncol; e += TF_THREADS) {
        const int r = j + 1 + e % nr, c = j + 1 + e / nr;
        A[r + (size_t)c * b] -= A[r + (size_t)j * b] * A[j + (size_t)c * b];
      }
      __syncthreads();
    }
    if (c1 < b) {
      // A[c0:c1, c1:b] <- L_ss^{-1} A[c0:c1, c1:b];  A[c1:b, c1:b] -= A[c1:b, c0:c1] A[c0:c1, c1:b]
      double* Lb = sm;
      double* buf = Lb + ib * ib;
      for (int e = tid; e < ib * ib; e += TF_THREADS) {
        const int r = e % ib, c = e / ib;
        Lb[e] = (r > c) ? A[c0 + r + (size_t)(c0 + c) * b] : 0.0;
      }
      __syncthreads();
      swap_solve(A + c0 + (size_t)c1 * b, b, nullptr, b, ib, b - c1, nullptr, nullptr, 0, Lb, buf,
                 SMEM_USER - ib * ib - 64);
      update_mn(sm, A + c1 + (size_t)c1 * b, b, A + c1 + (size_t)c0 * b, b, A + c0 + (size_t)c1 * b, b, b - c1,
                b - c1, ib);
      __syncthreads();
    }
  }
  for (int e = tid; e < b * b; e += TF_THREADS) {
    const int r = e % b, c = e / b;
    LX[e] = (r > c) ? A[e] : (r == c ? 1.0 : 0.0);
  }
  return first_zero;
}

// GESSM reference-blocked path: slab `item` of A_kj <- L_kk^{-1} P_kk A_kj.
__device__ inline void gessm_ref(const Ctx& cx, const double* LX, const int* ipiv, double* C, int item,
                                  double* sm) {
  const int b = cx.b, ib = cx.ib, tid = threadIdx.x;
  const int n0 = item * NS, nc = min(NS, b - n0);
  C += (size_t)n0 * b;
  // 1. P_kk: compose the b sequential interchanges into a gather permutation
  int* perm = reinterpret_cast<int*>(sm);
  double* buf = sm + (b + 1) / 2 + 1;
  for (int r = tid; r < b; r += TF_THREADS) perm[r] = r;
  __syncthreads();
  if (tid == 0)
    for (int j = 0; j < b; ++j) {
      const int r = ipiv[j] - 1;
      const int t = perm[j]; perm[j] = perm[r]; perm[r] = t;
    }
  __syncthreads();
  const int cap = SMEM_USER - (b + 1) / 2 - 8;
  const int cw = max(1, min(nc, cap / b));
  for (int cs = 0; cs < nc; cs += cw) {
    const int w = min(cw, nc - cs);
    for (int e = tid; e < b * w; e += TF_THREADS) buf[e] = ldg_cg(C + (size_t)cs * b + e);
    __syncthreads();
    for (int e = tid; e < b * w; e += TF_THREADS) {
      const int r = e % b, c = e / b;
      C[(size_t)cs * b + e] = buf[perm[r] + c * b];
    }
    __syncthreads();
  }
  // 2. blocked unit-lower forward solve
  for (int c0 = 0; c0 < b; c0 += ib) {
    const int c1 = c0 + ib;
    double* Lb = sm;
    for (int e = tid; e < ib * ib; e += TF_THREADS) {
      const int r = e % ib, c = e / ib;
      Lb[e] = (r > c) ? ldg_cg(LX + c0 + r + (size_t)(c0 + c) * b) : 0.0;
    }
    __syncthreads();
    swap_solve(C + c0, b, nullptr, b, ib, nc, nullptr, nullptr, 0, Lb, sm + ib * ib, SMEM_USER - ib * ib - 64);
    if (c1 < b) update_mn(sm, C + c1, b, LX + c1 + (size_t)c0 * b, b, C + c0, b, b - c1, nc, ib);
    __syncthreads();
  }
}

// Panel of DTSTRF (footnote PAPER.md:542-544): bottom P (b x ib, ld
// ldp), top Ub (ib x ib, ld ib, upper = U[c0:c1, c0:c1]), L-strip block Lsb (ld ib,
// zeroed), pivots piv[0..ib) (global, 1-based in [1, 2b]).  Returns first zero column.
__device__ inline int tstrf_panel(double* P, int ldp, int b, double* Ub, double* Lsb, int ib, int c0, int* piv,
                                  double* redv, int* redi, int nopiv) {
  const int tid = threadIdx.x;
  int first_zero = -1;
  for (int jj = 0; jj < ib; ++jj) {
    double v = -1.0;
    int idx = INT_MAX;
    if (tid == 0) { v = fabs(Ub[jj + jj * ib]); idx = -1; }
    for (int r = tid; r < (nopiv ? 0 : b); r += TF_THREADS) amax_merge(v, idx, fabs(P[r + (size_t)jj * ldp]), r);
    const int pr = block_amax(v, idx, redv, redi);
    if (pr >= 0) {
      for (int c = jj + tid; c < ib; c += TF_THREADS) {
        const double t = Ub[jj + c * ib];
        Ub[jj + c * ib] = P[pr + (size_t)c * ldp];
        P[pr + (size_t)c * ldp] = t;
      }
      for (int c = tid; c < jj; c += TF_THREADS) {
        const double t = Lsb[jj + c * ib];
        Lsb[jj + c * ib] = P[pr + (size_t)c * ldp];
        P[pr + (size_t)c * ldp] = t;
      }
    }
    if (tid == 0) piv[jj] = (pr >= 0) ? (b + pr + 1) : (c0 + jj + 1);
    __syncthreads();
    const double u = Ub[jj + jj * ib];
    if (u != 0.0) {
      for (int r = tid; r < b; r += TF_THREADS) P[r + (size_t)jj * ldp] = P[r + (size_t)jj * ldp] / u;
      __syncthreads();
      const int ncol = ib - jj - 1;
      for (int e = tid; e < b * ncol; e += TF_THREADS) {
        const int r = e % b, c = jj + 1 + e / b;
        P[r + (size_t)c * ldp] -= P[r + (size_t)jj * ldp] * Ub[jj + c * ib];
      }
    } else if (first_zero < 0) {
      first_zero = jj;
    }
    __syncthreads();
  }
  return first_zero;
}

// TSTRF: pairwise-pivoted LU of [U; A] (upper region of U only).
__device__ inline int tstrf_ref(const Ctx& cx, double* U, double* A, double* Ls, int* ipiv, double* sm) {
  const int b = cx.b, ib = cx.ib, tid = threadIdx.x;
  int first_zero = -1;
  for (int c0 = 0; c0 < b; c0 += ib) {
    const int c1 = c0 + ib;
    double* Ub = sm;
    double* Lsb = Ub + ib * ib;
    double* redv = Lsb + ib * ib;
    int* redi = reinterpret_cast<int*>(redv + TF_WARPS);
    double* P = redv + 2 * TF_WARPS;
    const bool in_smem = (size_t)b * ib + 2 * (size_t)ib * ib + 2 * TF_WARPS <= SMEM_USER;
    for (int e = tid; e < ib * ib; e += TF_THREADS) {
      const int r = e % ib, c = e / ib;
      Ub[e] = (r <= c) ? ldg_cg(U + c0 + r + (size_t)(c0 + c) * b) : 0.0;
      Lsb[e] = 0.0;
    }
    if (in_smem) {
      for (int e = tid; e < b * ib; e += TF_THREADS) P[e] = ldg_cg(A + (size_t)c0 * b + e);
    } else {
      P = A + (size_t)c0 * b;
    }
    __syncthreads();
    const int fz = tstrf_panel(P, b, b, Ub, Lsb, ib, c0, ipiv + c0, redv, redi, cx.nopiv);
    if (fz >= 0 && first_zero < 0) first_zero = c0 + fz;
    if (in_smem)
      for (int e = tid; e < b * ib; e += TF_THREADS) A[(size_t)c0 * b + e] = P[e];
    for (int e = tid; e < ib * ib; e += TF_THREADS) {
      const int r = e % ib, c = e / ib;
      if (r <= c) U[c0 + r + (size_t)(c0 + c) * b] = Ub[e];
      Ls[(size_t)c0 * ib + e] = Lsb[e];
    }
    __syncthreads();
    if (c1 < b) {
      // stage Lb = Lsb (strictly lower) at the front of smem, then swaps + (I+Ls)^{-1}
      double* Lb = sm;
      for (int e = tid; e < ib * ib; e += TF_THREADS) Lb[e] = ldg_cg(Ls + (size_t)c0 * ib + e);
      int* jslot = reinterpret_cast<int*>(Lb + ib * ib);
      int* srow = jslot + ib;
      int* snslot = srow + ib;
      int* rowslot = snslot + 2;
      __syncthreads();
      const int nslot = build_slots(ipiv, c0, ib, b, jslot, srow, rowslot, snslot);
      double* buf = Lb + ib * ib + (2 * ib + 2 + b + 1) / 2 + 2;
      const int cap = SMEM_USER - (int)(buf - sm);
      swap_solve(U + c0 + (size_t)c1 * b, b, A + (size_t)c1 * b, b, ib, b - c1, jslot, srow, nslot, Lb, buf, cap);
      update_mn(sm, A + (size_t)c1 * b, b, A + (size_t)c0 * b, b, U + c0 + (size_t)c1 * b, b, b, b - c1, ib);
      __syncthreads();
    }
  }
  return first_zero;
}

// SSSSM reference-blocked path: slab `item` of [U; A] <- L_ik^{-1} P_ik [U; A].
__device__ inline void ssssm_ref(const Ctx& cx, const double* L, const double* Ls, const int* ipiv, double* U,
                                  double* A, int item, double* sm) {
  const int b = cx.b, ib = cx.ib, tid = threadIdx.x;
  const int n0 = item * NS, nc = min(NS, b - n0);
  U += (size_t)n0 * b;
  A += (size_t)n0 * b;
  for (int c0 = 0; c0 < b; c0 += ib) {
    double* Lb = sm;
    for (int e = tid; e < ib * ib; e += TF_THREADS) Lb[e] = ldg_cg(Ls + (size_t)c0 * ib + e);
    int* jslot = reinterpret_cast<int*>(Lb + ib * ib);
    int* srow = jslot + ib;
    int* snslot = srow + ib;
    int* rowslot = snslot + 2;
    __syncthreads();
    const int nslot = build_slots(ipiv, c0, ib, b, jslot, srow, rowslot, snslot);
    double* buf = Lb + ib * ib + (2 * ib + 2 + b + 1) / 2 + 2;
    const int cap = SMEM_USER - (int)(buf - sm);
    swap_solve(U + c0, b, A, b, ib, nc, jslot, srow, nslot, Lb, buf, cap);
    update_mn(sm, A, b, L + (size_t)c0 * b, b, U + c0, b, b, nc, ib);
    __syncthreads();
  }
}

}  // namespace tf
#include "tf_lu_slab.cuh"
#include "tf_solve.cuh"
namespace tf {

TF_DEF_VARIANT(v_gessm_reg, gessm_reg, (Ctx cx, const double* LX, const int* ipiv, double* C, int item),
               (cx, LX, ipiv, C, item, dsm))
TF_DEF_VARIANT(v_ssssm_reg, ssssm_reg,
               (Ctx cx, const double* L, const double* Ls, const int* ipiv, double* U, double* A, int item),
               (cx, L, Ls, ipiv, U, A, item, dsm))
TF_DEF_VARIANT_RET(v_getrf_slab, getrf_slab, (Ctx cx, double* A, int* ipiv, double* LX, int cb, int ce),
                   (cx, A, ipiv, LX, cb, ce, dsm))
TF_DEF_VARIANT_RET(v_tstrf_slab, tstrf_slab,
                   (Ctx cx, double* U, double* A, double* Ls, int* ipiv, int cb, int ce, int bl, int bh, bool pnl),
                   (cx, U, A, Ls, ipiv, cb, ce, dsm, bl, bh, pnl))
TF_DEF_REF(v_gessm_ref, gessm_ref, (Ctx cx, const double* LX, const int* ipiv, double* C, int item),
           (cx, LX, ipiv, C, item, dsm))
TF_DEF_REF(v_ssssm_ref, ssssm_ref,
           (Ctx cx, const double* L, const double* Ls, const int* ipiv, double* U, double* A, int item),
           (cx, L, Ls, ipiv, U, A, item, dsm))
TF_DEF_REF_RET(v_getrf_ref, getrf_ref, (Ctx cx, double* A, int* ipiv, double* LX), (cx, A, ipiv, LX, dsm))
TF_DEF_REF_RET(v_tstrf_ref, tstrf_ref, (Ctx cx, double* U, double* A, double* Ls, int* ipiv), (cx, U, A, Ls, ipiv, dsm))

// LU update task kernels: register-slab path for b in {128, 256, 512}, ib in {32, 64}.
__device__ inline void gessm_item(const Ctx& cx, const double* LX, const int* ipiv, double* C, int item,
                                  double* sm) {
  if (ssrfb_reg_ok(cx.b, cx.ib)) TF_SLAB_DISPATCH(v_gessm_reg, cx, LX, ipiv, C, item);
  else v_gessm_ref(cx, LX, ipiv, C, item);
}
__device__ inline void ssssm_item(const Ctx& cx, const double* L, const double* Ls, const int* ipiv, double* U,
                                  double* A, int item, double* sm) {
  if (ssrfb_reg_ok(cx.b, cx.ib)) TF_SLAB_DISPATCH(v_ssssm_reg, cx, L, Ls, ipiv, U, A, item);
  else v_ssssm_ref(cx, L, Ls, ipiv, U, A, item);
}
// LU panel tasks: slab kernels for ib in {32, 64} (32-column slabs).
#define TF_SLAB_RET(fn, ...) (cx.b == 512 ? fn<4>(__VA_ARGS__) : cx.b == 256 ? fn<2>(__VA_ARGS__) : fn<1>(__VA_ARGS__))
__device__ inline int getrf_item(const Ctx& cx, double* A, int* ipiv, double* LX, double* sm) {
  if (ssrfb_reg_ok(cx.b, cx.ib)) return TF_SLAB_RET(v_getrf_slab, cx, A, ipiv, LX, 0, cx.b);
  return v_getrf_ref(cx, A, ipiv, LX);
}
// GETRF slab task of the slab-level DAG (returns the first zero-pivot local column or -1).
__device__ inline int getrf_slab_item(const Ctx& cx, double* A, int* ipiv, double* LX, int s, double* sm) {
  return TF_SLAB_RET(v_getrf_slab, cx, A, ipiv, LX, s * NSR, (s + 1) * NSR);
}
TF_DEF_REF(v_trsmu, trsmu_item, (Ctx cx, const double* U, double* X, int item), (cx, U, X, item, dsm))
TF_DEF_REF(v_xgemm, xgemm_item, (Ctx cx, const double* A, const double* B, double* C, int item),
           (cx, A, B, C, item, dsm))
TF_DEF_REF(v_unssssm, unssssm_item,
           (Ctx cx, const double* L, const double* Ls, const int* ipiv, double* X1, double* X2, int item),
           (cx, L, Ls, ipiv, X1, X2, item, dsm))
TF_DEF_REF(v_ungessm, ungessm_item, (Ctx cx, const double* F, const int* ipiv, double* X, int item),
           (cx, F, ipiv, X, item, dsm))

__device__ inline int tstrf_item(const Ctx& cx, double* U, double* A, double* Ls, int* ipiv, double* sm) {
  if (ssrfb_reg_ok(cx.b, cx.ib)) return TF_SLAB_RET(v_tstrf_slab, cx, U, A, Ls, ipiv, 0, cx.b, 0, INT_MAX, true);
  return v_tstrf_ref(cx, U, A, Ls, ipiv);
}
// TSTRF slab / apply tasks of the slab-level DAG: the older finished inner blocks [0, nfull - 1)
// by the apply task, the last one (and for ib = 64 the block's first slab) plus the panel by
// the slab task (nfull = finished inner blocks before slab s).
__device__ __forceinline__ int ts_nfull(int s, int ib) { return (s * NSR - (s * NSR) % ib) / ib; }
__device__ inline int tstrf_slab_item(const Ctx& cx, double* U, double* A, double* Ls, int* ipiv, int s, double* sm) {
  const int nf = ts_nfull(s, cx.ib);
  const int lo = ts_apply_split(true) && nf >= 2 ? nf - 1 : 0;
  return TF_SLAB_RET(v_tstrf_slab, cx, U, A, Ls, ipiv, s * NSR, (s + 1) * NSR, lo, INT_MAX, true);
}
__device__ inline void tstrf_apply_item(const Ctx& cx, double* U, double* A, double* Ls, int* ipiv, int s, double* sm) {
  const int nf = ts_nfull(s, cx.ib);
  (void)TF_SLAB_RET(v_tstrf_slab, cx, U, A, Ls, ipiv, s * NSR, (s + 1) * NSR, 0, nf - 1, false);
}

}  // namespace tf
