"""Pins of the oracle's solves and GENP (NEXT-3):

* GENP (Gaussian elimination with no pivoting): the unblocked textbook
  routine equals LAPACK's GEPP on column diagonally dominant matrices (GEPP then never
  swaps), and the tiled no-pivot Algorithm 3 equals the unblocked routine (any tiling of
  elimination without pivoting computes the same L and U) and equals pivoted Algorithm 3
  bitwise on the exact dyadic pin (no swaps there either).
* Solve with the Algorithm-3 factors, X <- U^{-1} N^{-1} X (Eq. eq:GETWPcompact): for
  b = n it is LAPACK's GEPP solve; on the exact dyadic pin with an integer solution it is
  exact; otherwise the backward error is small.
* Back substitution and the QR solve R^{-1} Q^T X against numpy's dense solve.
"""
import numpy as np
import scipy.linalg

import oracle
import tilegen


def _coldom(n, seed):
    A = tilegen.normal(n, seed)
    A[np.diag_indices(n)] = np.abs(A).sum(axis=0) + 1.0   # column diagonally dominant
    return A


def test_ref_genp_equals_gepp_on_diagonally_dominant():
    A = _coldom(48, 1)
    LU, info = oracle.ref_genp(A)
    lu, piv = scipy.linalg.lu_factor(A)
    assert info == 0 and np.array_equal(piv, np.arange(48))
    assert np.max(np.abs(LU - lu)) <= 1e-13 * np.max(np.abs(lu))


def test_tiled_genp_equals_unblocked():
    n, b, ib = 96, 32, 8
    A = _coldom(n, 2)
    F = oracle.pack(A, b)
    Ls, piv, info = oracle.lu_nopiv(F, n, b, ib)
    assert info == 0
    # U and the resulting N U = A identity (N = L for GENP)
    LU, _ = oracle.ref_genp(A)
    U_ref = np.triu(LU)
    U = oracle.lu_U(F, n, b)
    assert np.max(np.abs(U - U_ref)) <= 1e-12 * np.max(np.abs(U_ref))
    NU = oracle.lu_apply_N(F, Ls, piv, U, n, b, ib)
    assert np.linalg.norm(A - NU) / np.linalg.norm(A) <= 1e-14


def test_tiled_genp_pivots_are_identity_encodings():
    n, b, ib = 64, 16, 4
    A = tilegen.normal(n, 3)
    F = oracle.pack(A, b)
    _, piv, _ = oracle.lu_nopiv(F, n, b, ib)
    p = n // b
    for k in range(p):
        for i in range(k, p):
            o = (i + k * p) * b
            # GETRF keeps row j (j + 1 in [1, b]); TSTRF keeps the top row (j + 1, Z13)
            assert np.array_equal(piv[o:o + b], np.arange(b) + 1)


def test_genp_equals_getwp_on_exact_pin():
    n, b, ib = 64, 16, 4
    A, L0, U0 = tilegen.lu_exact(n, 3)
    F1 = oracle.pack(A, b)
    F2 = F1.copy()
    L1, p1, _ = oracle.lu(F1, n, b, ib)
    L2, p2, _ = oracle.lu_nopiv(F2, n, b, ib)
    assert np.array_equal(F1, F2) and np.array_equal(L1, L2) and np.array_equal(p1, p2)


def test_lu_solve_b_equals_n_is_lapack():
    n = 40
    A = tilegen.normal(n, 4)
    Y = tilegen.normal(n, 5)[:, :3]
    F = oracle.pack(A, n)
    Ls, piv, info = oracle.lu(F, n, n, 8)
    X = oracle.lu_solve(F, Ls, piv, Y, n, n, 8)
    Xl = scipy.linalg.lu_solve(scipy.linalg.lu_factor(A), Y)
    assert np.max(np.abs(X - Xl)) <= 1e-12 * np.max(np.abs(Xl))


def test_lu_solve_exact_pin():
    n, b, ib = 64, 16, 8
    A, L0, U0 = tilegen.lu_exact(n, 6)
    x0 = np.asfortranarray(np.arange(-8, 8, dtype=np.float64).reshape(-1, 1).repeat(4, axis=0)[:n])
    y = A @ x0                      # integer-valued, exact in binary64 (|y| < 2^53)
    F = oracle.pack(A, b)
    Ls, piv, _ = oracle.lu(F, n, b, ib)
    x = oracle.lu_solve(F, Ls, piv, y, n, b, ib)
    assert np.array_equal(x, x0)


def test_lu_solve_backward_error():
    n, b, ib = 256, 32, 8
    A = tilegen.normal(n, 7)
    y = tilegen.normal(n, 8)[:, :2]
    F = oracle.pack(A, b)
    Ls, piv, _ = oracle.lu(F, n, b, ib)
    x = oracle.lu_solve(F, Ls, piv, y, n, b, ib)
    be = np.max(np.abs(y - A @ x)) / (np.max(np.abs(A).sum(axis=1)) * np.max(np.abs(x)))
    assert be <= 1e-13, be
    assert np.max(np.abs(x - np.linalg.solve(A, y))) <= 1e-8 * np.max(np.abs(x))


def test_trsm_upper_and_qr_solve():
    n, b, ib = 96, 32, 8
    A = tilegen.uniform(n, 9)
    F = oracle.pack(A, b)
    T = oracle.qr(F, n, b, ib)
    y = tilegen.uniform(n, 10)[:, :3]
    x = oracle.qr_solve(F, T, y, n, b, ib)
    assert np.max(np.abs(x - np.linalg.solve(A, y))) <= 1e-10 * np.max(np.abs(x))
    R = oracle.qr_R(F, n, b)
    z = oracle.trsm_upper(F, R @ y, n, b)
    assert np.max(np.abs(z - y)) <= 1e-12 * np.max(np.abs(y))
    # integer upper-triangular R with power-of-two diagonal: back substitution is exact
    U = np.triu(np.round(tilegen.uniform(n, 11) * 8), 1) + np.diag(np.where(np.arange(n) % 2, 2.0, -4.0))
    U = np.asfortranarray(U)
    x0 = np.asfortranarray(np.ones((n, 1)))
    x = oracle.trsm_upper(oracle.pack(U, b), U @ x0, n, b)
    assert np.array_equal(x, x0)
