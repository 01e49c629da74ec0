/*
 * oracle.c — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load or call this library.  The product path (paper_0709_1272_b200/) never
 * links, imports or executes anything under oracle/, and this file shares no code,
 * header, table or helper with the CUDA path.
 *
 * What it is: a plain, slow, obviously-correct FP64 implementation of the three tiled
 * factorizations of the paper (arXiv 0709.1272, PAPER.md = /root/reference/PAPER.md):
 *   - Tiled Cholesky  — Algorithm 1 (alg:blkchol), kernels DPOTF2 /
 *     DTRSM / DGSMM.
 *   - Tiled QR        — Algorithm 2 (alg:blkqr), kernels DGEQRT /
 *     DLARFB / DTSQRT / DSSRFB with inner blocking s = ib
 *     (§3.2.3).
 *   - Tiled LU with incremental (tiled pairwise) pivoting — Algorithm 3 (alg:blklu,
 *     PAPER.md:560-576), kernels DGETRF / DGESSM / DTSTRF / DSSSSM,
 *     L-strip storage per the footnote at PAPER.md:542-544.
 * Every kernel is written in the order and notation of SURVEY.md §8(c) C1-C3 (the
 * readings of the paper this build adopts, listed in DESIGN.md §3).  Drivers run the
 * algorithms in program order; there is no blocking, fusion or reordering beyond what
 * the algorithm states.  Plain loops, no BLAS; compile with -O2 -ffp-contract=off so
 * that no FMA contraction changes the rounding of the written formulas.
 *
 * Also: brute-force references (unblocked Cholesky, unblocked Householder QR, GEPP,
 * GEWP) and the C4 checks (residuals, implicit application of Q and of N).
 *
 * Layout ("Block Data Layout"): p = n/b tiles per
 * side; tile (i,j) (0-based) starts at element (i + j*p)*b*b and is column-major
 * inside.  T strips (QR) and L strips (LU): strip (i,k) at (i + k*p)*ib*b, an
 * ib x b column-major block; inner block s occupies strip columns [s*ib, (s+1)*ib).
 * Pivots: int32, vector (i,k) at (i + k*p)*b, 1-based; GETRF in [1,b], TSTRF in
 * [1,2b] with bottom row r encoded as b+r+1.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OT(A, p, b, i, j) ((A) + ((size_t)(i) + (size_t)(j) * (size_t)(p)) * (size_t)(b) * (size_t)(b))
#define OE(X, ld, r, c) ((X)[(size_t)(r) + (size_t)(c) * (size_t)(ld)])
#define OSTRIP(S, p, b, ib, i, k) ((S) + ((size_t)(i) + (size_t)(k) * (size_t)(p)) * (size_t)(ib) * (size_t)(b))
#define OPIV(P, p, b, i, k) ((P) + ((size_t)(i) + (size_t)(k) * (size_t)(p)) * (size_t)(b))

/* ------------------------------------------------------------------------------------
 * Layout conversion (SPEC.md:41-56 from_dense / to_dense).  Dense is column-major m x n.
 * ---------------------------------------------------------------------------------- */
void o_pack(int64_t m, int64_t n, int64_t b, const double* dense, double* tiles) {
  int64_t p = m / b;
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = 0; r < m; ++r) {
      int64_t i = r / b, j = c / b;
      OE(OT(tiles, p, b, i, j), b, r % b, c % b) = OE(dense, m, r, c);
    }
}

void o_unpack(int64_t m, int64_t n, int64_t b, const double* tiles, double* dense) {
  int64_t p = m / b;
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = 0; r < m; ++r) {
      int64_t i = r / b, j = c / b;
      OE(dense, m, r, c) = OE(OT(tiles, p, b, i, j), b, r % b, c % b);
    }
}

/* ====================================================================================
 * C1 — Cholesky kernels
 * ================================================================================== */

/* DPOTF2: A_kk -> L_kk = chol(A_kk), lower, positive diagonal
 * ("unit" at PAPER.md:262 read as an erratum).  Reads/writes the lower
 * triangle only; the strict upper triangle is never touched (Z2).
 * Returns 0, or the 1-based local column whose pivot d is not > 0 (LAPACK info, Z3). */
int o_potrf(int64_t b, double* A) {
  for (int64_t j = 0; j < b; ++j) {
    double d = OE(A, b, j, j);
    for (int64_t m = 0; m < j; ++m) d -= OE(A, b, j, m) * OE(A, b, j, m);
    if (!(d > 0.0)) return (int)(j + 1);
    double ljj = sqrt(d);
    OE(A, b, j, j) = ljj;
    for (int64_t r = j + 1; r < b; ++r) {
      double s = OE(A, b, r, j);
      for (int64_t m = 0; m < j; ++m) s -= OE(A, b, r, m) * OE(A, b, j, m);
      OE(A, b, r, j) = s / ljj;
    }
  }
  return 0;
}

/* DTRSM: L_ik = A_ik L_kk^{-T}; row by row,
 * X[r,c] = (A[r,c] - sum_{m<c} X[r,m] L[c,m]) / L[c,c]. */
void o_trsm(int64_t b, const double* L, double* A) {
  for (int64_t r = 0; r < b; ++r)
    for (int64_t c = 0; c < b; ++c) {
      double s = OE(A, b, r, c);
      for (int64_t m = 0; m < c; ++m) s -= OE(A, b, r, m) * OE(L, b, c, m);
      OE(A, b, r, c) = s / OE(L, b, c, c);
    }
}

/* DGSMM, diagonal case ("take advantage of their triangular
 * structure"): C -= A A^T on the lower triangle only (SYRK; Z2). */
void o_syrk(int64_t b, const double* A, double* C) {
  for (int64_t c = 0; c < b; ++c)
    for (int64_t r = c; r < b; ++r) {
      double s = OE(C, b, r, c);
      for (int64_t m = 0; m < b; ++m) s -= OE(A, b, r, m) * OE(A, b, c, m);
      OE(C, b, r, c) = s;
    }
}

/* DGSMM, off-diagonal case: C -= A B^T. */
void o_gemm_nt(int64_t b, const double* A, const double* B, double* C) {
  for (int64_t c = 0; c < b; ++c)
    for (int64_t r = 0; r < b; ++r) {
      double s = OE(C, b, r, c);
      for (int64_t m = 0; m < b; ++m) s -= OE(A, b, r, m) * OE(B, b, c, m);
      OE(C, b, r, c) = s;
    }
}

/* Algorithm 1 in program order.  Returns 0 or the first failing
 * global column (1-based); on failure stops writing (Z3). */
int o_chol(int64_t n, int64_t b, double* A) {
  int64_t p = n / b;
  for (int64_t k = 0; k < p; ++k) {
    int info = o_potrf(b, OT(A, p, b, k, k));
    if (info) return (int)(k * b + info);
    for (int64_t i = k + 1; i < p; ++i) o_trsm(b, OT(A, p, b, k, k), OT(A, p, b, i, k));
    for (int64_t i = k + 1; i < p; ++i)
      for (int64_t j = k + 1; j <= i; ++j) {
        if (i == j) o_syrk(b, OT(A, p, b, i, k), OT(A, p, b, i, i));
        else o_gemm_nt(b, OT(A, p, b, i, k), OT(A, p, b, j, k), OT(A, p, b, i, j));
      }
  }
  return 0;
}

/* ====================================================================================
 * C2 — QR kernels (inner blocking §3.2.3)
 * ================================================================================== */

/* House(alpha, x): LAPACK dlarfg semantics without the safmin rescaling loop (Z6).
 * On return x holds v, *alpha holds beta; returns tau. */
static double o_house(double* alpha, double* x, int64_t len, int64_t stride) {
  double ss = 0.0;
  for (int64_t r = 0; r < len; ++r) ss += x[r * stride] * x[r * stride];
  double xn = sqrt(ss);
  if (xn == 0.0) {
    return 0.0; /* tau = 0, beta = alpha, v = x = 0 */
  }
  double a = *alpha;
  double nrm = sqrt(a * a + xn * xn);
  double beta = (a >= 0.0) ? -nrm : nrm;
  double tau = (beta - a) / beta;
  double den = a - beta;
  for (int64_t r = 0; r < len; ++r) x[r * stride] = x[r * stride] / den;
  *alpha = beta;
  return tau;
}

/* T_s column jj of the forward columnwise compact-WY factor (dlarft):
 * T[jj,jj] = tau_j, T[0:jj,jj] = T[0:jj,0:jj] * w with w = -tau_j * (V[:,c0:j]^T v_j).
 * `w` is passed in (already holding V^T v_j); Ts is ib x ib, column-major ld ib. */
static void o_tcol(double* Ts, int64_t ib, int64_t jj, double tau, double* w) {
  for (int64_t m = 0; m < jj; ++m) w[m] = -tau * w[m];
  for (int64_t r = 0; r < jj; ++r) {
    double s = 0.0;
    for (int64_t m = r; m < jj; ++m) s += OE(Ts, ib, r, m) * w[m];
    OE(Ts, ib, r, jj) = s;
  }
  OE(Ts, ib, jj, jj) = tau;
  for (int64_t r = jj + 1; r < ib; ++r) OE(Ts, ib, r, jj) = 0.0;
}

/* Element (r, m) of the unit-lower reflector block V_s of a GEQRT'ed tile, rows
 * counted in the tile: 1 on the diagonal (r == c0+m), the stored v below, 0 above. */
static double o_vgeq(const double* A, int64_t b, int64_t c0, int64_t r, int64_t m) {
  int64_t c = c0 + m;
  if (r < c) return 0.0;
  if (r == c) return 1.0;
  return OE(A, b, r, c);
}

/* Apply the block reflector of inner block s of GEQRT'ed tile V (T strip Tst) to
 * rows c0..b-1 of C (b x ncol, ld ldc): C <- (I - V_s op(T_s) V_s^T) C with
 * op = T^T when trans != 0 (the factorization, Q^T), op = T when trans == 0 (Q). */
static void o_apply_geq_block(int64_t b, int64_t ib, int64_t s, const double* V, const double* Tst,
                              double* C, int64_t ldc, int64_t ncol, int trans) {
  int64_t c0 = s * ib;
  const double* Ts = Tst + (size_t)c0 * ib;
  double* W = (double*)malloc(sizeof(double) * ib * (ncol > 0 ? ncol : 1));
  double* W2 = (double*)malloc(sizeof(double) * ib * (ncol > 0 ? ncol : 1));
  for (int64_t c = 0; c < ncol; ++c)
    for (int64_t m = 0; m < ib; ++m) {
      double acc = 0.0;
      for (int64_t r = c0; r < b; ++r) acc += o_vgeq(V, b, c0, r, m) * OE(C, ldc, r, c);
      OE(W, ib, m, c) = acc;
    }
  for (int64_t c = 0; c < ncol; ++c)
    for (int64_t m = 0; m < ib; ++m) {
      double acc = 0.0;
      for (int64_t q = 0; q < ib; ++q)
        acc += (trans ? OE(Ts, ib, q, m) : OE(Ts, ib, m, q)) * OE(W, ib, q, c);
      OE(W2, ib, m, c) = acc;
    }
  for (int64_t c = 0; c < ncol; ++c)
    for (int64_t r = c0; r < b; ++r) {
      double acc = 0.0;
      for (int64_t m = 0; m < ib; ++m) acc += o_vgeq(V, b, c0, r, m) * OE(W2, ib, m, c);
      OE(C, ldc, r, c) -= acc;
    }
  free(W);
  free(W2);
}

/* DGEQRT with inner block ib: A -> (V strict lower, R upper,
 * T strip).  C2: per inner block, panel Householder, T_s (dlarft), trailing update. */
void o_geqrt(int64_t b, int64_t ib, double* A, double* Tst) {
  double* w = (double*)malloc(sizeof(double) * ib);
  for (int64_t s = 0; s * ib < b; ++s) {
    int64_t c0 = s * ib, c1 = c0 + ib;
    double* Ts = Tst + (size_t)c0 * ib;
    for (int64_t j = c0; j < c1; ++j) {
      double tau = o_house(&OE(A, b, j, j), &OE(A, b, j + 1, j), b - j - 1, 1);
      /* apply H_j = I - tau [1;v][1;v]^T to A[j:b, j+1:c1] */
      for (int64_t c = j + 1; c < c1; ++c) {
        double wc = OE(A, b, j, c);
        for (int64_t r = j + 1; r < b; ++r) wc += OE(A, b, r, j) * OE(A, b, r, c);
        OE(A, b, j, c) -= tau * wc;
        for (int64_t r = j + 1; r < b; ++r) OE(A, b, r, c) -= tau * wc * OE(A, b, r, j);
      }
      /* T_s column: w[m] = V[:, c0+m]^T v_j over rows >= j */
      int64_t jj = j - c0;
      for (int64_t m = 0; m < jj; ++m) {
        double acc = OE(A, b, j, c0 + m); /* v_j has 1 at row j */
        for (int64_t r = j + 1; r < b; ++r) acc += OE(A, b, r, c0 + m) * OE(A, b, r, j);
        w[m] = acc;
      }
      o_tcol(Ts, ib, jj, tau, w);
    }
    if (c1 < b) o_apply_geq_block(b, ib, s, A, Tst, &OE(A, b, 0, c1), b, b - c1, 1);
  }
  free(w);
}

/* DLARFB: A_kj <- Q_kk^T A_kj, i.e. (I - V_s T_s^T V_s^T) for
 * s = 0..t-1 in order (reading Z5). */
void o_larfb(int64_t b, int64_t ib, const double* V, const double* Tst, double* C) {
  for (int64_t s = 0; s * ib < b; ++s) o_apply_geq_block(b, ib, s, V, Tst, C, b, b, 1);
}

/* Block reflector of a TSQRT'ed pair: top rows c0..c1-1 of X1 (identity part of V),
 * bottom all b rows of X2 (dense V_s = Vb[:, c0:c1]).
 * trans != 0: X <- (I - V T^T V^T) X, else (I - V T V^T) X. */
static void o_apply_ts_block(int64_t b, int64_t ib, int64_t s, const double* Vb, const double* Tst,
                             double* X1, int64_t ld1, double* X2, int64_t ld2, int64_t ncol,
                             int trans) {
  int64_t c0 = s * ib;
  const double* Ts = Tst + (size_t)c0 * ib;
  double* W = (double*)malloc(sizeof(double) * ib * (ncol > 0 ? ncol : 1));
  double* W2 = (double*)malloc(sizeof(double) * ib * (ncol > 0 ? ncol : 1));
  for (int64_t c = 0; c < ncol; ++c)
    for (int64_t m = 0; m < ib; ++m) {
      double acc = OE(X1, ld1, c0 + m, c);
      for (int64_t r = 0; r < b; ++r) acc += OE(Vb, b, r, c0 + m) * OE(X2, ld2, r, c);
      OE(W, ib, m, c) = acc;
    }
  for (int64_t c = 0; c < ncol; ++c)
    for (int64_t m = 0; m < ib; ++m) {
      double acc = 0.0;
      for (int64_t q = 0; q < ib; ++q)
        acc += (trans ? OE(Ts, ib, q, m) : OE(Ts, ib, m, q)) * OE(W, ib, q, c);
      OE(W2, ib, m, c) = acc;
    }
  for (int64_t c = 0; c < ncol; ++c) {
    for (int64_t m = 0; m < ib; ++m) OE(X1, ld1, c0 + m, c) -= OE(W2, ib, m, c);
    for (int64_t r = 0; r < b; ++r) {
      double acc = 0.0;
      for (int64_t m = 0; m < ib; ++m) acc += OE(Vb, b, r, c0 + m) * OE(W2, ib, m, c);
      OE(X2, ld2, r, c) -= acc;
    }
  }
  free(W);
  free(W2);
}

/* DTSQRT (inner blocking PAPER.md:637-647): QR of [R; A] with R the
 * upper triangle of the diagonal tile (only its upper region is read or written) and
 * A a full tile; A <- V_ik (top part implicitly identity), T strip written. */
void o_tsqrt(int64_t b, int64_t ib, double* R, double* A, double* Tst) {
  double* w = (double*)malloc(sizeof(double) * ib);
  for (int64_t s = 0; s * ib < b; ++s) {
    int64_t c0 = s * ib, c1 = c0 + ib;
    double* Ts = Tst + (size_t)c0 * ib;
    for (int64_t j = c0; j < c1; ++j) {
      double tau = o_house(&OE(R, b, j, j), &OE(A, b, 0, j), b, 1);
      for (int64_t c = j + 1; c < c1; ++c) {
        double wc = OE(R, b, j, c);
        for (int64_t r = 0; r < b; ++r) wc += OE(A, b, r, j) * OE(A, b, r, c);
        OE(R, b, j, c) -= tau * wc;
        for (int64_t r = 0; r < b; ++r) OE(A, b, r, c) -= tau * wc * OE(A, b, r, j);
      }
      int64_t jj = j - c0;
      for (int64_t m = 0; m < jj; ++m) {
        double acc = 0.0; /* top parts e_{c0+m}, e_j are orthogonal */
        for (int64_t r = 0; r < b; ++r) acc += OE(A, b, r, c0 + m) * OE(A, b, r, j);
        w[m] = acc;
      }
      o_tcol(Ts, ib, jj, tau, w);
    }
    if (c1 < b) o_apply_ts_block(b, ib, s, A, Tst, &OE(R, b, 0, c1), b, &OE(A, b, 0, c1), b, b - c1, 1);
  }
  free(w);
}

/* DSSRFB: [R_kj; A_ij] <- Q_ik^T [R_kj; A_ij],
 * inner blocks s = 0..t-1 in order. */
void o_ssrfb(int64_t b, int64_t ib, const double* V, const double* Tst, double* R, double* A) {
  for (int64_t s = 0; s * ib < b; ++s) o_apply_ts_block(b, ib, s, V, Tst, R, b, A, b, b, 1);
}

/* Algorithm 2, square p x p tiles, in program order. */
/* Algorithm 2 on an m x n matrix of p x q tiles ("the tiled QR of
 * a p-by-q tiled matrix"), k < min(p, q).  T strips (i,k) at (i + k*p)*ib*b. */
void o_qr_mn(int64_t m, int64_t n, int64_t b, int64_t ib, double* A, double* T) {
  int64_t p = m / b, q = n / b, kk = p < q ? p : q;
  for (int64_t k = 0; k < kk; ++k) {
    o_geqrt(b, ib, OT(A, p, b, k, k), OSTRIP(T, p, b, ib, k, k));
    for (int64_t j = k + 1; j < q; ++j)
      o_larfb(b, ib, OT(A, p, b, k, k), OSTRIP(T, p, b, ib, k, k), OT(A, p, b, k, j));
    for (int64_t i = k + 1; i < p; ++i) {
      o_tsqrt(b, ib, OT(A, p, b, k, k), OT(A, p, b, i, k), OSTRIP(T, p, b, ib, i, k));
      for (int64_t j = k + 1; j < q; ++j)
        o_ssrfb(b, ib, OT(A, p, b, i, k), OSTRIP(T, p, b, ib, i, k), OT(A, p, b, k, j), OT(A, p, b, i, j));
    }
  }
}

/* Algorithm 2, square p x p tiles, program order. */
void o_qr(int64_t n, int64_t b, int64_t ib, double* A, double* T) { o_qr_mn(n, n, b, ib, A, T); }

/* C4: X (n x ncol, column-major, ld n) <- Q X (trans == 0) or Q^T X (trans != 0),
 * Q the orthogonal factor held implicitly by the factored tiles and T strips.
 * Q X applies the inverses of the factorization's block reflectors in reverse task
 * order and reverse inner-block order, with T untransposed. */
void o_qr_apply_mn(int64_t m, int64_t n, int64_t b, int64_t ib, const double* F, const double* T, double* X,
                   int64_t ncol, int trans) {
  /* m x n factors (p x q tiles): Q is m x m, X is m x ncol (ld m) */
  int64_t p = m / b, q = n / b, t = b / ib, kk = p < q ? p : q;
  if (trans) {
    for (int64_t k = 0; k < kk; ++k) {
      for (int64_t s = 0; s < t; ++s)
        o_apply_geq_block(b, ib, s, OT(F, p, b, k, k), OSTRIP(T, p, b, ib, k, k), X + k * b, m, ncol, 1);
      for (int64_t i = k + 1; i < p; ++i)
        for (int64_t s = 0; s < t; ++s)
          o_apply_ts_block(b, ib, s, OT(F, p, b, i, k), OSTRIP(T, p, b, ib, i, k), X + k * b, m,
                           X + i * b, m, ncol, 1);
    }
  } else {
    for (int64_t k = kk - 1; k >= 0; --k) {
      for (int64_t i = p - 1; i > k; --i)
        for (int64_t s = t - 1; s >= 0; --s)
          o_apply_ts_block(b, ib, s, OT(F, p, b, i, k), OSTRIP(T, p, b, ib, i, k), X + k * b, m,
                           X + i * b, m, ncol, 0);
      for (int64_t s = t - 1; s >= 0; --s)
        o_apply_geq_block(b, ib, s, OT(F, p, b, k, k), OSTRIP(T, p, b, ib, k, k), X + k * b, m, ncol, 0);
    }
  }
}

void o_qr_apply(int64_t n, int64_t b, int64_t ib, const double* F, const double* T, double* X,
                int64_t ncol, int trans) {
  o_qr_apply_mn(n, n, b, ib, F, T, X, ncol, trans);
}

/* ====================================================================================
 * C3 — LU kernels (storage PAPER.md:536-546 and footnote)
 * ================================================================================== */

static void o_swap_rows(double* X, int64_t ld, int64_t r1, int64_t r2, int64_t c0, int64_t c1) {
  if (r1 == r2) return;
  for (int64_t c = c0; c < c1; ++c) {
    double tmp = OE(X, ld, r1, c);
    OE(X, ld, r1, c) = OE(X, ld, r2, c);
    OE(X, ld, r2, c) = tmp;
  }
}

/* Pivoting switch for GENP (Gaussian elimination with no pivoting):
 * when set, o_getrf keeps row j and o_tstrf keeps the top row for every column; the
 * arithmetic is otherwise that of Algorithm 3.  Only o_lu_nopiv sets it. */
static int o_nopiv = 0;

/* Pivot-decision recorder — test instrumentation for the C5 seed-margin reading
 * (DESIGN.md §3): when armed, every pivot decision of o_getrf /
 * o_tstrf appends (|winner|, |runner-up|) in program order.  It only reads the
 * candidates after the decision; the arithmetic is unchanged whether armed or not. */
static double* o_dec = NULL;
static int64_t o_dec_cap = 0, o_dec_n = 0;
void o_decisions_arm(double* buf, int64_t cap) { o_dec = buf; o_dec_cap = cap; o_dec_n = 0; }
int64_t o_decisions_count(void) { return o_dec_n; }
static void o_dec_push(double best, double second) {
  if (o_dec && o_dec_n < o_dec_cap) { o_dec[2 * o_dec_n] = best; o_dec[2 * o_dec_n + 1] = second; }
  if (o_dec) ++o_dec_n;
}

/* DGETRF: P A = L U with partial pivoting inside the tile, LAPACK
 * dgetrf semantics with block ib (Z12: whole-tile-row swaps).  First argmax of fabs
 * over rows j..b-1 (idamax rule, Z11).  *info gets the first zero-pivot local column
 * (1-based) if none recorded yet. */
void o_getrf(int64_t b, int64_t ib, double* A, int32_t* ipiv, int* info) {
  for (int64_t s = 0; s * ib < b; ++s) {
    int64_t c0 = s * ib, c1 = c0 + ib;
    for (int64_t j = c0; j < c1; ++j) {
      int64_t r = j;
      double best = fabs(OE(A, b, j, j));
      for (int64_t rr = j + 1; rr < b && !o_nopiv; ++rr)
        if (fabs(OE(A, b, rr, j)) > best) { best = fabs(OE(A, b, rr, j)); r = rr; }
      if (o_dec) {
        double second = -1.0;
        for (int64_t rr = j; rr < b; ++rr)
          if (rr != r && fabs(OE(A, b, rr, j)) > second) second = fabs(OE(A, b, rr, j));
        o_dec_push(best, second);
      }
      ipiv[j] = (int32_t)(r + 1);
      if (OE(A, b, r, j) != 0.0) {
        o_swap_rows(A, b, j, r, 0, b);
        for (int64_t rr = j + 1; rr < b; ++rr) OE(A, b, rr, j) /= OE(A, b, j, j);
      } else if (*info == 0) {
        *info = (int)(j + 1);
      }
      for (int64_t c = j + 1; c < c1; ++c)
        for (int64_t rr = j + 1; rr < b; ++rr) OE(A, b, rr, c) -= OE(A, b, rr, j) * OE(A, b, j, c);
    }
    if (c1 < b) {
      /* A[c0:c1, c1:b] <- L_ss^{-1} A[c0:c1, c1:b] (unit lower) */
      for (int64_t c = c1; c < b; ++c)
        for (int64_t r = c0; r < c1; ++r) {
          double acc = OE(A, b, r, c);
          for (int64_t m = c0; m < r; ++m) acc -= OE(A, b, r, m) * OE(A, b, m, c);
          OE(A, b, r, c) = acc;
        }
      /* A[c1:b, c1:b] -= A[c1:b, c0:c1] A[c0:c1, c1:b] */
      for (int64_t c = c1; c < b; ++c)
        for (int64_t r = c1; r < b; ++r) {
          double acc = OE(A, b, r, c);
          for (int64_t m = c0; m < c1; ++m) acc -= OE(A, b, r, m) * OE(A, b, m, c);
          OE(A, b, r, c) = acc;
        }
    }
  }
}

/* DGESSM: A_kj <- L_kk^{-1} P_kk A_kj — all swaps, then the blocked
 * unit-lower forward solve. */
void o_gessm(int64_t b, int64_t ib, const double* L, const int32_t* ipiv, double* A) {
  for (int64_t j = 0; j < b; ++j) o_swap_rows(A, b, j, ipiv[j] - 1, 0, b);
  for (int64_t s = 0; s * ib < b; ++s) {
    int64_t c0 = s * ib, c1 = c0 + ib;
    for (int64_t c = 0; c < b; ++c)
      for (int64_t r = c0; r < c1; ++r) {
        double acc = OE(A, b, r, c);
        for (int64_t m = c0; m < r; ++m) acc -= OE(L, b, r, m) * OE(A, b, m, c);
        OE(A, b, r, c) = acc;
      }
    for (int64_t c = 0; c < b; ++c)
      for (int64_t r = c1; r < b; ++r) {
        double acc = OE(A, b, r, c);
        for (int64_t m = c0; m < c1; ++m) acc -= OE(L, b, r, m) * OE(A, b, m, c);
        OE(A, b, r, c) = acc;
      }
  }
}

/* DTSTRF (footnote PAPER.md:542-544): pairwise-pivoted LU of [U; A]
 * with U the upper triangle of the diagonal tile (only its upper region is touched),
 * A a full tile.  A <- bottom multipliers, Ls strip <- the t unit-lower ib x ib blocks
 * (strictly lower part stored), ipiv in [1,2b].  Reading C3 / Z10 / Z11 / Z13. */
void o_tstrf(int64_t b, int64_t ib, double* U, double* A, double* Ls, int32_t* ipiv, int* info) {
  for (int64_t s = 0; s * ib < b; ++s) {
    int64_t c0 = s * ib, c1 = c0 + ib;
    for (int64_t c = c0; c < c1; ++c)
      for (int64_t r = 0; r < ib; ++r) OE(Ls, ib, r, c) = 0.0;
    for (int64_t j = c0; j < c1; ++j) {
      int64_t r = -1;
      double best = fabs(OE(U, b, j, j));
      for (int64_t rr = 0; rr < b && !o_nopiv; ++rr)
        if (fabs(OE(A, b, rr, j)) > best) { best = fabs(OE(A, b, rr, j)); r = rr; }
      if (o_dec) {
        double second = (r >= 0) ? fabs(OE(U, b, j, j)) : -1.0;
        for (int64_t rr = 0; rr < b; ++rr)
          if (rr != r && fabs(OE(A, b, rr, j)) > second) second = fabs(OE(A, b, rr, j));
        o_dec_push(best, second);
      }
      if (r >= 0) {
        ipiv[j] = (int32_t)(b + r + 1);
        for (int64_t c = j; c < c1; ++c) {
          double tmp = OE(U, b, j, c); OE(U, b, j, c) = OE(A, b, r, c); OE(A, b, r, c) = tmp;
        }
        for (int64_t c = c0; c < j; ++c) {
          double tmp = OE(Ls, ib, j - c0, c); OE(Ls, ib, j - c0, c) = OE(A, b, r, c); OE(A, b, r, c) = tmp;
        }
      } else {
        ipiv[j] = (int32_t)(j + 1);
      }
      if (OE(U, b, j, j) != 0.0) {
        for (int64_t rr = 0; rr < b; ++rr) OE(A, b, rr, j) /= OE(U, b, j, j);
        for (int64_t c = j + 1; c < c1; ++c)
          for (int64_t rr = 0; rr < b; ++rr) OE(A, b, rr, c) -= OE(A, b, rr, j) * OE(U, b, j, c);
      } else if (*info == 0) {
        *info = (int)(j + 1);
      }
    }
    if (c1 < b) {
      for (int64_t j = c0; j < c1; ++j)
        if (ipiv[j] > b) {
          int64_t r = ipiv[j] - b - 1;
          for (int64_t c = c1; c < b; ++c) {
            double tmp = OE(U, b, j, c); OE(U, b, j, c) = OE(A, b, r, c); OE(A, b, r, c) = tmp;
          }
        }
      for (int64_t c = c1; c < b; ++c)
        for (int64_t r = c0; r < c1; ++r) {
          double acc = OE(U, b, r, c);
          for (int64_t m = c0; m < r; ++m) acc -= OE(Ls, ib, r - c0, m) * OE(U, b, m, c);
          OE(U, b, r, c) = acc;
        }
      for (int64_t c = c1; c < b; ++c)
        for (int64_t r = 0; r < b; ++r) {
          double acc = OE(A, b, r, c);
          for (int64_t m = c0; m < c1; ++m) acc -= OE(A, b, r, m) * OE(U, b, m, c);
          OE(A, b, r, c) = acc;
        }
    }
  }
}

/* DSSSSM: [U_kj; A_ij] <- L_ik^{-1} P_ik [U_kj; A_ij] per inner block:
 * swaps of whole rows, (I+Ls_s)^{-1} on the top rows, then A_ij -= L_ik[:,s] U_kj[s,:]. */
void o_ssssm(int64_t b, int64_t ib, const double* L, const double* Ls, const int32_t* ipiv,
             double* U, double* A) {
  for (int64_t s = 0; s * ib < b; ++s) {
    int64_t c0 = s * ib, c1 = c0 + ib;
    for (int64_t j = c0; j < c1; ++j)
      if (ipiv[j] > b) {
        int64_t r = ipiv[j] - b - 1;
        for (int64_t c = 0; c < b; ++c) {
          double tmp = OE(U, b, j, c); OE(U, b, j, c) = OE(A, b, r, c); OE(A, b, r, c) = tmp;
        }
      }
    for (int64_t c = 0; c < b; ++c)
      for (int64_t r = c0; r < c1; ++r) {
        double acc = OE(U, b, r, c);
        for (int64_t m = c0; m < r; ++m) acc -= OE(Ls, ib, r - c0, m) * OE(U, b, m, c);
        OE(U, b, r, c) = acc;
      }
    for (int64_t c = 0; c < b; ++c)
      for (int64_t r = 0; r < b; ++r) {
        double acc = OE(A, b, r, c);
        for (int64_t m = c0; m < c1; ++m) acc -= OE(L, b, r, m) * OE(U, b, m, c);
        OE(A, b, r, c) = acc;
      }
  }
}

/* Algorithm 3, square p x p tiles, program order.  Returns 0 or the
 * smallest global column (1-based) whose pivot was exactly zero. */
int o_lu_mn(int64_t m, int64_t n, int64_t b, int64_t ib, double* A, double* Ls, int32_t* ipiv) {
  /* Algorithm 3 on an m x n matrix of p x q tiles, k < min(p, q) */
  int64_t p = m / b, q = n / b, kk = p < q ? p : q;
  int64_t best = 0;
  for (int64_t k = 0; k < kk; ++k) {
    int info = 0;
    o_getrf(b, ib, OT(A, p, b, k, k), OPIV(ipiv, p, b, k, k), &info);
    if (info && (best == 0 || k * b + info < best)) best = k * b + info;
    for (int64_t j = k + 1; j < q; ++j)
      o_gessm(b, ib, OT(A, p, b, k, k), OPIV(ipiv, p, b, k, k), OT(A, p, b, k, j));
    for (int64_t i = k + 1; i < p; ++i) {
      info = 0;
      o_tstrf(b, ib, OT(A, p, b, k, k), OT(A, p, b, i, k), OSTRIP(Ls, p, b, ib, i, k),
              OPIV(ipiv, p, b, i, k), &info);
      if (info && (best == 0 || k * b + info < best)) best = k * b + info;
      for (int64_t j = k + 1; j < q; ++j)
        o_ssssm(b, ib, OT(A, p, b, i, k), OSTRIP(Ls, p, b, ib, i, k), OPIV(ipiv, p, b, i, k),
                OT(A, p, b, k, j), OT(A, p, b, i, j));
    }
  }
  return (int)best;
}

int o_lu(int64_t n, int64_t b, int64_t ib, double* A, double* Ls, int32_t* ipiv) {
  return o_lu_mn(n, n, b, ib, A, Ls, ipiv);
}

/* GENP in tiled form: Algorithm 3 with every pivot kept (o_nopiv).
 * Pivots come out as the identity encodings (j + 1). */
int o_lu_nopiv(int64_t n, int64_t b, int64_t ib, double* A, double* Ls, int32_t* ipiv) {
  o_nopiv = 1;
  int info = o_lu(n, b, ib, A, Ls, ipiv);
  o_nopiv = 0;
  return info;
}

/* X (n x ncol, ld ldx) <- U^{-1} X with U the upper triangle of the BDL matrix F (tiles
 * j >= i; R of Algorithm 2 or U of Algorithm 3): textbook back substitution, row by row
 * from the bottom, x[r] = (x[r] - sum_{m>r} U[r,m] x[m]) / U[r,r]. */
void o_trsm_upper_bdl(int64_t n, int64_t b, const double* F, double* X, int64_t ncol, int64_t ldx) {
  int64_t p = n / b;
  for (int64_t c = 0; c < ncol; ++c)
    for (int64_t r = n - 1; r >= 0; --r) {
      double acc = OE(X, ldx, r, c);
      for (int64_t m = r + 1; m < n; ++m)
        acc -= OE(OT(F, p, b, r / b, m / b), b, r % b, m % b) * OE(X, ldx, m, c);
      OE(X, ldx, r, c) = acc / OE(OT(F, p, b, r / b, r / b), b, r % b, r % b);
    }
}

/* Solve with the factors of Algorithm 3 (Eq. eq:GETWPcompact, N U = A):
 * X <- A^{-1} X = U^{-1} N^{-1} X.  N^{-1} X applies the elimination steps to X in program
 * order — for each k the DGESSM step on tile row k (all swaps, then the blocked unit-lower
 * solve), then for i > k the DSSSSM step on tile rows (k, i) (per inner block: swaps,
 * (I + Ls_s)^{-1} on the top rows, bottom -= L_ik[:, s] top) — exactly the operations the
 * factorization applies to the columns right of panel k (C3); then back substitution. */
void o_lu_solve(int64_t n, int64_t b, int64_t ib, const double* F, const double* Ls, const int32_t* ipiv,
                double* X, int64_t ncol, int64_t ldx) {
  int64_t p = n / b;
  for (int64_t k = 0; k < p; ++k) {
    double* xk = X + k * b;
    const double* Lkk = OT(F, p, b, k, k);
    const int32_t* pk = OPIV(ipiv, p, b, k, k);
    for (int64_t j = 0; j < b; ++j) o_swap_rows(xk, ldx, j, pk[j] - 1, 0, ncol);
    for (int64_t s = 0; s * ib < b; ++s) {
      int64_t c0 = s * ib, c1 = c0 + ib;
      for (int64_t c = 0; c < ncol; ++c)
        for (int64_t r = c0; r < c1; ++r) {
          double acc = OE(xk, ldx, r, c);
          for (int64_t m = c0; m < r; ++m) acc -= OE(Lkk, b, r, m) * OE(xk, ldx, m, c);
          OE(xk, ldx, r, c) = acc;
        }
      for (int64_t c = 0; c < ncol; ++c)
        for (int64_t r = c1; r < b; ++r) {
          double acc = OE(xk, ldx, r, c);
          for (int64_t m = c0; m < c1; ++m) acc -= OE(Lkk, b, r, m) * OE(xk, ldx, m, c);
          OE(xk, ldx, r, c) = acc;
        }
    }
    for (int64_t i = k + 1; i < p; ++i) {
      double* xi = X + i * b;
      const double* L = OT(F, p, b, i, k);
      const double* Lst = OSTRIP(Ls, p, b, ib, i, k);
      const int32_t* pv = OPIV(ipiv, p, b, i, k);
      for (int64_t s = 0; s * ib < b; ++s) {
        int64_t c0 = s * ib, c1 = c0 + ib;
        for (int64_t j = c0; j < c1; ++j)
          if (pv[j] > b) {
            int64_t r = pv[j] - b - 1;
            for (int64_t c = 0; c < ncol; ++c) {
              double tmp = OE(xk, ldx, j, c); OE(xk, ldx, j, c) = OE(xi, ldx, r, c); OE(xi, ldx, r, c) = tmp;
            }
          }
        for (int64_t c = 0; c < ncol; ++c)
          for (int64_t r = c0; r < c1; ++r) {
            double acc = OE(xk, ldx, r, c);
            for (int64_t m = c0; m < r; ++m) acc -= OE(Lst, ib, r - c0, m) * OE(xk, ldx, m, c);
            OE(xk, ldx, r, c) = acc;
          }
        for (int64_t c = 0; c < ncol; ++c)
          for (int64_t r = 0; r < b; ++r) {
            double acc = OE(xi, ldx, r, c);
            for (int64_t m = c0; m < c1; ++m) acc -= OE(L, b, r, m) * OE(xk, ldx, m, c);
            OE(xi, ldx, r, c) = acc;
          }
      }
    }
  }
  o_trsm_upper_bdl(n, b, F, X, ncol, ldx);
}

/* C4 / Eq. (eq:formula N), (eq:GETWPcompact):
 * X (n x ncol, ld n) <- N X, N = (prod of the elementary L and P of GETWP)^{-1},
 * applied implicitly by undoing every elimination step in reverse program order. */
void o_lu_apply_N_mn(int64_t m, int64_t n, int64_t b, int64_t ib, const double* F, const double* Ls,
                     const int32_t* ipiv, double* X, int64_t ncol) {
  /* m x n factors (p x q tiles): N is m x m, X is m x ncol (ld m) */
  int64_t p = m / b, q = n / b, t = b / ib, kk = p < q ? p : q;
  const int64_t ldn = m;
  for (int64_t k = kk - 1; k >= 0; --k) {
    double* x1 = X + k * b;
    for (int64_t i = p - 1; i > k; --i) {
      const double* L = OT(F, p, b, i, k);
      const double* Lst = OSTRIP(Ls, p, b, ib, i, k);
      const int32_t* pv = OPIV(ipiv, p, b, i, k);
      double* x2 = X + i * b;
      for (int64_t s = t - 1; s >= 0; --s) {
        int64_t c0 = s * ib, c1 = c0 + ib;
        for (int64_t c = 0; c < ncol; ++c) {
          /* x2 += L[:, c0:c1] x1[c0:c1] (uses x1 before its update) */
          for (int64_t r = 0; r < b; ++r) {
            double acc = 0.0;
            for (int64_t m = c0; m < c1; ++m) acc += OE(L, b, r, m) * OE(x1, ldn, m, c);
            OE(x2, ldn, r, c) += acc;
          }
          /* x1[c0:c1] <- (I + Ls_s) x1[c0:c1]; rows descending so inputs stay original */
          for (int64_t r = c1 - 1; r >= c0; --r) {
            double acc = 0.0;
            for (int64_t m = c0; m < r; ++m) acc += OE(Lst, ib, r - c0, m) * OE(x1, ldn, m, c);
            OE(x1, ldn, r, c) += acc;
          }
        }
        for (int64_t j = c1 - 1; j >= c0; --j)
          if (pv[j] > b) {
            int64_t r = pv[j] - b - 1;
            for (int64_t c = 0; c < ncol; ++c) {
              double tmp = OE(x1, ldn, j, c); OE(x1, ldn, j, c) = OE(x2, ldn, r, c); OE(x2, ldn, r, c) = tmp;
            }
          }
      }
    }
    /* undo GETRF(k): x <- L_kk x (unit lower, full tile), then undo swaps in reverse */
    const double* Lkk = OT(F, p, b, k, k);
    const int32_t* pv = OPIV(ipiv, p, b, k, k);
    for (int64_t c = 0; c < ncol; ++c)
      for (int64_t r = b - 1; r >= 0; --r) {
        double acc = 0.0;
        for (int64_t m = 0; m < r; ++m) acc += OE(Lkk, b, r, m) * OE(x1, ldn, m, c);
        OE(x1, ldn, r, c) += acc;
      }
    for (int64_t j = b - 1; j >= 0; --j) {
      int64_t r = pv[j] - 1;
      if (r != j)
        for (int64_t c = 0; c < ncol; ++c) {
          double tmp = OE(x1, ldn, j, c); OE(x1, ldn, j, c) = OE(x1, ldn, r, c); OE(x1, ldn, r, c) = tmp;
        }
    }
  }
}

void o_lu_apply_N(int64_t n, int64_t b, int64_t ib, const double* F, const double* Ls,
                  const int32_t* ipiv, double* X, int64_t ncol) {
  o_lu_apply_N_mn(n, n, b, ib, F, Ls, ipiv, X, ncol);
}

/* ====================================================================================
 * Brute-force references (SURVEY §8(c) C5 "Brute force for n <= 64", "Special cases")
 * Dense column-major n x n.
 * ================================================================================== */

/* Unblocked right-looking scalar Cholesky (textbook).  Lower triangle. */
int o_ref_chol(int64_t n, double* A) {
  for (int64_t k = 0; k < n; ++k) {
    double d = OE(A, n, k, k);
    if (!(d > 0.0)) return (int)(k + 1);
    OE(A, n, k, k) = sqrt(d);
    for (int64_t i = k + 1; i < n; ++i) OE(A, n, i, k) /= OE(A, n, k, k);
    for (int64_t j = k + 1; j < n; ++j)
      for (int64_t i = j; i < n; ++i) OE(A, n, i, j) -= OE(A, n, i, k) * OE(A, n, j, k);
  }
  return 0;
}

/* Unblocked Householder QR (dgeqr2): R upper, v below the diagonal, tau[n]. */
void o_ref_qr(int64_t n, double* A, double* tau) {
  for (int64_t j = 0; j < n; ++j) {
    tau[j] = o_house(&OE(A, n, j, j), &OE(A, n, j + 1, j), n - j - 1, 1);
    for (int64_t c = j + 1; c < n; ++c) {
      double wc = OE(A, n, j, c);
      for (int64_t r = j + 1; r < n; ++r) wc += OE(A, n, r, j) * OE(A, n, r, c);
      OE(A, n, j, c) -= tau[j] * wc;
      for (int64_t r = j + 1; r < n; ++r) OE(A, n, r, c) -= tau[j] * wc * OE(A, n, r, j);
    }
  }
}

/* Unblocked GEPP (dgetf2): ipiv 1-based, L strictly lower, U upper.  Returns info. */
int o_ref_gepp(int64_t n, double* A, int32_t* ipiv) {
  int info = 0;
  for (int64_t j = 0; j < n; ++j) {
    int64_t r = j;
    double best = fabs(OE(A, n, j, j));
    for (int64_t rr = j + 1; rr < n; ++rr)
      if (fabs(OE(A, n, rr, j)) > best) { best = fabs(OE(A, n, rr, j)); r = rr; }
    ipiv[j] = (int32_t)(r + 1);
    if (OE(A, n, r, j) != 0.0) {
      o_swap_rows(A, n, j, r, 0, n);
      for (int64_t rr = j + 1; rr < n; ++rr) OE(A, n, rr, j) /= OE(A, n, j, j);
    } else if (!info) {
      info = (int)(j + 1);
    }
    for (int64_t c = j + 1; c < n; ++c)
      for (int64_t rr = j + 1; rr < n; ++rr) OE(A, n, rr, c) -= OE(A, n, rr, j) * OE(A, n, j, c);
  }
  return info;
}

/* GENP — Gaussian elimination with no pivoting, unblocked textbook
 * right-looking form: L strictly lower (multipliers), U upper.  Returns info (first zero
 * pivot, 1-based). */
int o_ref_genp(int64_t n, double* A) {
  int info = 0;
  for (int64_t j = 0; j < n; ++j) {
    if (OE(A, n, j, j) != 0.0) {
      for (int64_t rr = j + 1; rr < n; ++rr) OE(A, n, rr, j) /= OE(A, n, j, j);
    } else if (!info) {
      info = (int)(j + 1);
    }
    for (int64_t c = j + 1; c < n; ++c)
      for (int64_t rr = j + 1; rr < n; ++rr) OE(A, n, rr, c) -= OE(A, n, rr, j) * OE(A, n, j, c);
  }
  return info;
}

/* GEWP — Gaussian elimination with pairwise pivoting (Wilkinson):
 * for each column k, rows i = k+1..n-1 in order: row k and row i compete, the larger
 * |entry| becomes row k (strictly greater wins), then row i -= l * row k with
 * l = A[i,k]/A[k,k] stored in A[i,k].  swapped[k + i*n] = 1 when rows were exchanged. */
int o_ref_gewp(int64_t n, double* A, int32_t* swapped) {
  int info = 0;
  for (int64_t k = 0; k < n; ++k)
    for (int64_t i = k + 1; i < n; ++i) {
      swapped[k + i * n] = 0;
      if (fabs(OE(A, n, i, k)) > fabs(OE(A, n, k, k))) {
        o_swap_rows(A, n, k, i, k, n);
        swapped[k + i * n] = 1;
      }
      if (OE(A, n, k, k) != 0.0) {
        double l = OE(A, n, i, k) / OE(A, n, k, k);
        OE(A, n, i, k) = l;
        for (int64_t c = k + 1; c < n; ++c) OE(A, n, i, c) -= l * OE(A, n, k, c);
      } else if (!info) {
        info = (int)(k + 1);
      }
    }
  return info;
}

/* ====================================================================================
 * Checks (C4)
 * ================================================================================== */

/* ||A - L L^T||_F / ||A||_F over the full symmetric A, where A_lo holds the lower
 * triangle of A and L the factor, both dense column-major n x n. */
double o_chol_residual(int64_t n, const double* A_lo, const double* L) {
  double num = 0.0, den = 0.0;
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = c; r < n; ++r) {
      double acc = 0.0;
      for (int64_t m = 0; m <= c; ++m) acc += OE(L, n, r, m) * OE(L, n, c, m);
      double a = OE(A_lo, n, r, c);
      double e = a - acc;
      double wgt = (r == c) ? 1.0 : 2.0;
      num += wgt * e * e;
      den += wgt * a * a;
    }
  return sqrt(num) / sqrt(den);
}

/* Leading-order flop counts of the two update kernels whose costs the paper states
 * (PAPER.md:655-656 DSSRFB 4b^3 + s b^2, PAPER.md:674 DSSSSM 2b^3 + s b^2; reading Z7).
 * The other kinds have no printed count and are not provided (NaN). */
double o_kernel_flops(int kind, double b, double s) {
  switch (kind) {
    case 7: return 4.0 * b * b * b + s * b * b;        /* SSRFB */
    case 11: return 2.0 * b * b * b + s * b * b;       /* SSSSM */
    default: return NAN;
  }
}


/* ====================================================================================
 * Host multicore baseline: the oracle's tile kernels under a thread-pool DAG executor —
 * the paper's runtime (§4.1): a shared progress table (in-degree
 * counters), every thread repeatedly takes the highest-priority ready task (kind ranks
 * panel > couple-factor > row-update > couple-update; ties by program
 * order) and releases its successors when done.  Dependencies come from each task's
 * read / write sets over tiles, with diagonal tiles of QR / LU split into the V / L
 * (strictly lower) and R / U (upper) regions (TSQRT / TSTRF touch only the upper one).
 * Every tile's updates keep their program order, so the result is bitwise that of the
 * sequential drivers.  Reported as a baseline only (bench.py cpu_baseline).
 * ================================================================================== */
typedef struct { int kind, k, i, j; } OTask;
typedef struct {
  int alg; int64_t n, b, ib, p;
  double *A, *aux; int32_t* ipiv;
  OTask* t; int nt;
  int *indeg, *soff, *succ, *level;
  int *heap; int nheap;            /* ready tasks, min (level, index) */
  int done, abort_, info;
  pthread_mutex_t mu; pthread_cond_t cv;
} OPool;

static int o_key_less(const OPool* P, int a, int b) {
  return P->level[a] != P->level[b] ? P->level[a] < P->level[b] : a < b;
}
static void o_heap_push(OPool* P, int x) {
  int c = P->nheap++;
  P->heap[c] = x;
  while (c > 0) {
    int par = (c - 1) / 2;
    if (!o_key_less(P, P->heap[c], P->heap[par])) break;
    int t = P->heap[c]; P->heap[c] = P->heap[par]; P->heap[par] = t; c = par;
  }
}
static int o_heap_pop(OPool* P) {
  int top = P->heap[0];
  P->heap[0] = P->heap[--P->nheap];
  int c = 0;
  for (;;) {
    int l = 2 * c + 1, r = l + 1, m = c;
    if (l < P->nheap && o_key_less(P, P->heap[l], P->heap[m])) m = l;
    if (r < P->nheap && o_key_less(P, P->heap[r], P->heap[m])) m = r;
    if (m == c) break;
    int t = P->heap[c]; P->heap[c] = P->heap[m]; P->heap[m] = t; c = m;
  }
  return top;
}

static void o_run_task(OPool* P, const OTask* T) {
  int64_t p = P->p, b = P->b, ib = P->ib;
  double* A = P->A;
  int k = T->k, i = T->i, j = T->j, info = 0;
  switch (T->kind) {
    case 0: info = o_potrf(b, OT(A, p, b, k, k)); if (info) info += (int)(k * b); break;
    case 1: o_trsm(b, OT(A, p, b, k, k), OT(A, p, b, i, k)); break;
    case 2: o_syrk(b, OT(A, p, b, i, k), OT(A, p, b, i, i)); break;
    case 3: o_gemm_nt(b, OT(A, p, b, i, k), OT(A, p, b, j, k), OT(A, p, b, i, j)); break;
    case 4: o_geqrt(b, ib, OT(A, p, b, k, k), OSTRIP(P->aux, p, b, ib, k, k)); break;
    case 5: o_larfb(b, ib, OT(A, p, b, k, k), OSTRIP(P->aux, p, b, ib, k, k), OT(A, p, b, k, j)); break;
    case 6: o_tsqrt(b, ib, OT(A, p, b, k, k), OT(A, p, b, i, k), OSTRIP(P->aux, p, b, ib, i, k)); break;
    case 7: o_ssrfb(b, ib, OT(A, p, b, i, k), OSTRIP(P->aux, p, b, ib, i, k), OT(A, p, b, k, j), OT(A, p, b, i, j)); break;
    case 8: o_getrf(b, ib, OT(A, p, b, k, k), OPIV(P->ipiv, p, b, k, k), &info); if (info) info += (int)(k * b); break;
    case 9: o_gessm(b, ib, OT(A, p, b, k, k), OPIV(P->ipiv, p, b, k, k), OT(A, p, b, k, j)); break;
    case 10:
      o_tstrf(b, ib, OT(A, p, b, k, k), OT(A, p, b, i, k), OSTRIP(P->aux, p, b, ib, i, k), OPIV(P->ipiv, p, b, i, k), &info);
      if (info) info += (int)(k * b);
      break;
    case 11:
      o_ssssm(b, ib, OT(A, p, b, i, k), OSTRIP(P->aux, p, b, ib, i, k), OPIV(P->ipiv, p, b, i, k), OT(A, p, b, k, j),
              OT(A, p, b, i, j));
      break;
  }
  if (info) {
    pthread_mutex_lock(&P->mu);
    if (!P->info || info < P->info) P->info = info;
    if (T->kind == 0) P->abort_ = 1;  /* Cholesky stops at the first failure (Z3) */
    pthread_mutex_unlock(&P->mu);
  }
}

static void* o_worker(void* arg) {
  OPool* P = (OPool*)arg;
  pthread_mutex_lock(&P->mu);
  for (;;) {
    while (P->nheap == 0 && P->done < P->nt && !P->abort_) pthread_cond_wait(&P->cv, &P->mu);
    if (P->abort_ || P->done >= P->nt) break;
    int t = o_heap_pop(P);
    pthread_mutex_unlock(&P->mu);
    o_run_task(P, &P->t[t]);
    pthread_mutex_lock(&P->mu);
    P->done++;
    for (int e = P->soff[t]; e < P->soff[t + 1]; ++e)
      if (--P->indeg[P->succ[e]] == 0) o_heap_push(P, P->succ[e]);
    pthread_cond_broadcast(&P->cv);
  }
  pthread_cond_broadcast(&P->cv);
  pthread_mutex_unlock(&P->mu);
  return NULL;
}

/* alg 0 chol, 1 qr, 2 lu; aux = T / L strips, ipiv (LU).  Returns info. */
int o_factor_par(int alg, int64_t n, int64_t b, int64_t ib, double* A, double* aux, int32_t* ipiv, int nthreads) {
  int64_t p = n / b;
  int64_t cap = alg == 0 ? p * (p + 1) * (p + 2) / 6 + p * p : p * (p + 1) * (2 * p + 1) / 6 + p * p;
  OTask* t = (OTask*)malloc(sizeof(OTask) * cap);
  int nt = 0;
  if (alg == 0) {
    for (int k = 0; k < p; ++k) {
      t[nt++] = (OTask){0, k, k, k};
      for (int i = k + 1; i < p; ++i) t[nt++] = (OTask){1, k, i, k};
      for (int i = k + 1; i < p; ++i)
        for (int j = k + 1; j <= i; ++j) t[nt++] = (OTask){i == j ? 2 : 3, k, i, j};
    }
  } else {
    int F = alg == 1 ? 4 : 8;
    for (int k = 0; k < p; ++k) {
      t[nt++] = (OTask){F, k, k, k};
      for (int j = k + 1; j < p; ++j) t[nt++] = (OTask){F + 1, k, k, j};
      for (int i = k + 1; i < p; ++i) {
        t[nt++] = (OTask){F + 2, k, i, k};
        for (int j = k + 1; j < p; ++j) t[nt++] = (OTask){F + 3, k, i, j};
      }
    }
  }
  /* resources: tile (i,j) region r -> 2*(i + j*p) + r (r = 1: upper region of a diagonal
   * tile in QR / LU); strip + pivots (i,k) -> 2*p*p + i + k*p */
  int64_t nres = 3 * p * p;
  int* lastw = (int*)malloc(sizeof(int) * nres);
  int** rd = (int**)calloc(nres, sizeof(int*));
  int* nrd = (int*)calloc(nres, sizeof(int));
  int* crd = (int*)calloc(nres, sizeof(int));
  for (int64_t x = 0; x < nres; ++x) lastw[x] = -1;
  int* pcnt = (int*)calloc(nt, sizeof(int));
  int pcap = 16 * nt + 16;
  int* pl = (int*)malloc(sizeof(int) * pcap);  /* (task, pred) pairs */
  int np = 0;
  int* level = (int*)malloc(sizeof(int) * nt);
#define TILE(a, c, r) (2 * ((int64_t)(a) + (int64_t)(c) * p) + (r))
#define STRIP_(a, c) (2 * p * p + (int64_t)(a) + (int64_t)(c) * p)
  for (int x = 0; x < nt; ++x) {
    const OTask* T = &t[x];
    int64_t rs[6], ws[6];
    int nr = 0, nw = 0;
    int k = T->k, i = T->i, j = T->j;
    switch (T->kind) {
      case 0: ws[nw++] = TILE(k, k, 0); break;
      case 1: rs[nr++] = TILE(k, k, 0); ws[nw++] = TILE(i, k, 0); break;
      case 2: rs[nr++] = TILE(i, k, 0); ws[nw++] = TILE(i, i, 0); break;
      case 3: rs[nr++] = TILE(i, k, 0); rs[nr++] = TILE(j, k, 0); ws[nw++] = TILE(i, j, 0); break;
      case 4: case 8: ws[nw++] = TILE(k, k, 0); ws[nw++] = TILE(k, k, 1); ws[nw++] = STRIP_(k, k); break;
      case 5: case 9: rs[nr++] = TILE(k, k, 0); rs[nr++] = STRIP_(k, k); ws[nw++] = TILE(k, j, 0); break;
      case 6: case 10: ws[nw++] = TILE(k, k, 1); ws[nw++] = TILE(i, k, 0); ws[nw++] = STRIP_(i, k); break;
      default:  /* 7, 11: reads (i,k) + strip, writes (k,j) and (i,j) (both regions if diagonal) */
        rs[nr++] = TILE(i, k, 0); rs[nr++] = STRIP_(i, k);
        ws[nw++] = TILE(k, j, 0);
        ws[nw++] = TILE(i, j, 0);
        if (i == j) ws[nw++] = TILE(i, j, 1);
        break;
    }
    switch (T->kind) {
      case 0: case 4: case 8: level[x] = 0; break;
      case 1: case 6: case 10: level[x] = 1; break;
      case 5: case 9: level[x] = 2; break;
      default: level[x] = 3;
    }
#define ADDP(q) do { if ((q) >= 0 && (q) != x) { if (np == pcap) { pcap *= 2; pl = (int*)realloc(pl, sizeof(int) * pcap); } pl[np++] = (q); pcnt[x]++; } } while (0)
    for (int a = 0; a < nr; ++a) {
      ADDP(lastw[rs[a]]);
      if (nrd[rs[a]] == crd[rs[a]]) { crd[rs[a]] = crd[rs[a]] ? 2 * crd[rs[a]] : 4; rd[rs[a]] = (int*)realloc(rd[rs[a]], sizeof(int) * crd[rs[a]]); }
      rd[rs[a]][nrd[rs[a]]++] = x;
    }
    for (int a = 0; a < nw; ++a) {
      ADDP(lastw[ws[a]]);
      for (int r = 0; r < nrd[ws[a]]; ++r) ADDP(rd[ws[a]][r]);
      nrd[ws[a]] = 0;
      lastw[ws[a]] = x;
    }
#undef ADDP
  }
#undef TILE
#undef STRIP_
  /* pl holds preds grouped by task in order; build successor CSR (duplicates harmless:
   * each duplicate edge is counted once in indeg and once in succ) */
  int* indeg = (int*)calloc(nt, sizeof(int));
  int* soff = (int*)calloc(nt + 1, sizeof(int));
  { int q = 0; for (int x = 0; x < nt; ++x) for (int c = 0; c < pcnt[x]; ++c, ++q) { soff[pl[q] + 1]++; indeg[x]++; } }
  for (int x = 0; x < nt; ++x) soff[x + 1] += soff[x];
  int* succ = (int*)malloc(sizeof(int) * (np + 1));
  int* fill = (int*)malloc(sizeof(int) * (nt + 1));
  memcpy(fill, soff, sizeof(int) * (nt + 1));
  { int q = 0; for (int x = 0; x < nt; ++x) for (int c = 0; c < pcnt[x]; ++c, ++q) succ[fill[pl[q]]++] = x; }
  OPool P;
  memset(&P, 0, sizeof(P));
  P.alg = alg; P.n = n; P.b = b; P.ib = ib; P.p = p; P.A = A; P.aux = aux; P.ipiv = ipiv;
  P.t = t; P.nt = nt; P.indeg = indeg; P.soff = soff; P.succ = succ; P.level = level;
  P.heap = (int*)malloc(sizeof(int) * (nt + 1));
  pthread_mutex_init(&P.mu, NULL);
  pthread_cond_init(&P.cv, NULL);
  for (int x = 0; x < nt; ++x)
    if (indeg[x] == 0) o_heap_push(&P, x);
  if (nthreads < 1) nthreads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  for (int w = 0; w < nthreads; ++w) pthread_create(&th[w], NULL, o_worker, &P);
  for (int w = 0; w < nthreads; ++w) pthread_join(th[w], NULL);
  int info = P.info;
  pthread_mutex_destroy(&P.mu);
  pthread_cond_destroy(&P.cv);
  for (int64_t x = 0; x < nres; ++x) free(rd[x]);
  free(rd); free(nrd); free(crd); free(lastw); free(pcnt); free(pl); free(level); free(indeg); free(soff);
  free(succ); free(fill); free(P.heap); free(th); free(t);
  return info;
}
