"""Pins of the oracle's rectangular tiled QR / LU: Algorithm 2 on an
m x n matrix of p x q tiles and Algorithm 3 likewise.

* QR: R^T R = A^T A (R = Q^T A with Q orthogonal; independent of how Q is represented),
  |diag R| equal to LAPACK's QR of the same matrix, and A = Q R through the oracle's own
  compact-WY application; the square case equals o_qr bitwise.
* LU: one tile row (p = 1, b = m) is GEPP on the m x n matrix = LAPACK getrf (pivots
  identical, factors to rounding); N U = A for p > 1 (Eq. eq:GETWPcompact); |multipliers|
  <= 1; the square case equals o_lu bitwise.
"""
import numpy as np
import pytest
import scipy.linalg

import oracle
import tilegen


def _mat(m, n, seed, gen=tilegen.uniform):
    return np.asfortranarray(gen(max(m, n), seed)[:m, :n])


@pytest.mark.parametrize("m,n,b,ib", [(96, 48, 16, 4), (48, 96, 16, 8), (128, 32, 32, 8), (64, 64, 16, 4),
                                      (160, 96, 32, 16)])
def test_qr_mn(m, n, b, ib):
    A = _mat(m, n, 1)
    F = oracle.pack(A, b)
    T = oracle.qr_mn(F, m, n, b, ib)
    R = oracle.upper_mn(F, m, n, b)
    k = min(m, n)
    assert np.linalg.norm(R.T @ R - A.T @ A) <= 1e-14 * np.linalg.norm(A.T @ A) * max(m, n)
    Rl = np.linalg.qr(A, mode="r")
    assert np.allclose(np.abs(np.diag(R[:k, :k])), np.abs(np.diag(Rl[:k, :k])), rtol=1e-12, atol=0)
    QR = oracle.qr_apply_mn(F, T, np.vstack([R[:k], np.zeros((m - k, n))]) if m > k else R[:k], m, n, b, ib)
    assert np.linalg.norm(QR - A) <= 1e-14 * np.linalg.norm(A) * max(m, n)
    if m == n:
        F2 = oracle.pack(A, b)
        T2 = oracle.qr(F2, n, b, ib)
        assert np.array_equal(F, F2) and np.array_equal(T, T2)


@pytest.mark.parametrize("m,n,ib", [(32, 64, 8), (48, 96, 16)])
def test_lu_mn_one_tile_row_is_gepp(m, n, ib):
    A = _mat(m, n, 2, tilegen.normal)
    # one tile row and b = m requires n % m == 0 for BDL; use q tiles of width b = m
    if n % m:
        pytest.skip("BDL needs b | n")
    F = oracle.pack(A, m)
    Ls, piv, info = oracle.lu_mn(F, m, n, m, ib)
    lu, pl = scipy.linalg.lu_factor(A[:, :m])
    assert np.array_equal(piv[:m] - 1, pl)


@pytest.mark.parametrize("m,n,b,ib", [(96, 48, 16, 4), (48, 96, 16, 8), (128, 32, 32, 8), (64, 128, 32, 32),
                                      (64, 64, 16, 4)])
def test_lu_mn_identity_and_multipliers(m, n, b, ib):
    A = _mat(m, n, 3, tilegen.normal)
    F = oracle.pack(A, b)
    Ls, piv, info = oracle.lu_mn(F, m, n, b, ib)
    assert info == 0
    U = oracle.upper_mn(F, m, n, b)
    NU = oracle.lu_apply_N_mn(F, Ls, piv, U, m, n, b, ib)
    assert np.linalg.norm(A - NU) / np.linalg.norm(A) <= 1e-13
    # stored multipliers bounded by 1: below the diagonal of the tiles
    # of block column k < min(p, q)
    D = oracle.unpack(F, m, n, b)
    k = min(m, n)
    assert np.max(np.abs(np.tril(D[:, :k], -1))) <= 1.0
    if m == n:
        F2 = oracle.pack(A, b)
        L2, p2, _ = oracle.lu(F2, n, b, ib)
        assert np.array_equal(F, F2) and np.array_equal(Ls, L2) and np.array_equal(piv, p2)


def test_gepp_wide_tile_row():
    """p = 1 (b = m) on a wide m x 2m matrix: the first tile is GEPP (LAPACK pivots), and
    the second tile column receives L^{-1} P (GESSM) = LAPACK's U12."""
    m = 32
    A = _mat(m, 2 * m, 4, tilegen.normal)
    F = oracle.pack(A, m)
    Ls, piv, info = oracle.lu_mn(F, m, 2 * m, m, 8)
    P, L, U = scipy.linalg.lu(A)   # A = P L U (LAPACK GEPP on the whole wide matrix)
    D = oracle.unpack(F, m, 2 * m, m)
    assert np.max(np.abs(np.triu(D) - U)) <= 1e-12 * np.max(np.abs(U))
