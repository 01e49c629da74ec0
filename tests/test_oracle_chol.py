"""Pins of the oracle's tiled Cholesky (Algorithm 1) against things
other than itself: exact integer factors, LAPACK (numpy), the textbook right-looking
scalar algorithm (b = 1), and the SPEC worked example."""
import numpy as np
import pytest

import oracle
import tilegen


def _factor(A, b):
    n = A.shape[0]
    F = oracle.pack(A, b)
    info = oracle.chol(F, n, b)
    return F, info


@pytest.mark.parametrize("n,b,seed", [(64, 16, 0), (96, 32, 1), (40, 8, 2), (48, 48, 3), (30, 5, 4)])
def test_exact_integer_pin(n, b, seed):
    """A = L0 L0^T with integer L0 (diag in {1,2,4}) => L = L0 bitwise."""
    A, L0 = tilegen.chol_exact(n, seed)
    F, info = _factor(A, b)
    assert info == 0
    L = oracle.tile_lower_L(F, n, b)
    assert np.array_equal(L, L0)


@pytest.mark.parametrize("n,b", [(64, 16), (48, 12), (33, 11)])
def test_vs_lapack(n, b):
    A = tilegen.spd(n, 7)
    F, info = _factor(A, b)
    assert info == 0
    L = oracle.tile_lower_L(F, n, b)
    Lref = np.linalg.cholesky(A)
    assert np.max(np.abs(L - Lref)) <= 1e-14 * np.max(np.abs(Lref))


def test_b1_equals_right_looking_scalar_bitwise():
    """b = 1: every task is a scalar op, so the tiled run IS the right-looking scalar
    algorithm (same operations, same order) — bitwise."""
    n = 24
    A = tilegen.spd(n, 3)
    F, info = _factor(A, 1)
    Lref, info2 = oracle.ref_chol(A)
    assert info == 0 and info2 == 0
    assert np.array_equal(oracle.tile_lower_L(F, n, 1), np.tril(Lref))


def test_unblocked_ref_vs_lapack():
    """Pins the brute-force reference itself."""
    A = tilegen.spd(50, 11)
    L, info = oracle.ref_chol(A)
    assert info == 0
    assert np.max(np.abs(np.tril(L) - np.linalg.cholesky(A))) <= 1e-13


def test_residual_config1_shape():
    """||A - L L^T||_F/||A||_F <= 1e-13 (BASELINE north_star) on the config-1 recipe."""
    n, b = 256, 32
    A = tilegen.spd(n, 0)
    F, info = _factor(A, b)
    assert info == 0
    L = oracle.tile_lower_L(F, n, b)
    res = np.linalg.norm(A - L @ L.T) / np.linalg.norm(A)
    assert res <= 1e-13
    # the oracle's own residual routine agrees with numpy's
    assert abs(oracle.chol_residual(np.tril(A), L) - res) <= 1e-16


def test_spec_potf2_example():
    """[[4,2],[2,5]] -> [[2,0],[1,2]]; strict upper untouched (Z2)."""
    A = np.asfortranarray([[4.0, 2.0], [2.0, 5.0]])
    assert oracle.potrf(A) == 0
    assert A[0, 0] == 2 and A[1, 0] == 1 and A[1, 1] == 2 and A[0, 1] == 2.0


def test_spec_trsm_example():
    """l = 2I, a = [[2,4],[6,8]] -> [[1,2],[3,4]]."""
    L = np.asfortranarray(2.0 * np.eye(2))
    A = np.asfortranarray([[2.0, 4.0], [6.0, 8.0]])
    oracle.trsm(L, A)
    assert np.array_equal(A, [[1.0, 2.0], [3.0, 4.0]])


def test_gemm_syrk_vs_numpy():
    r = np.random.default_rng(5)
    b = 12
    A = np.asfortranarray(r.standard_normal((b, b)))
    B = np.asfortranarray(r.standard_normal((b, b)))
    C = np.asfortranarray(r.standard_normal((b, b)))
    C1 = C.copy(order="F")
    oracle.gemm_nt(A, B, C1)
    assert np.allclose(C1, C - A @ B.T, atol=1e-13, rtol=0)
    C2 = C.copy(order="F")
    oracle.syrk(A, C2)
    ref = C - A @ A.T
    assert np.allclose(np.tril(C2), np.tril(ref), atol=1e-13, rtol=0)
    assert np.array_equal(np.triu(C2, 1), np.triu(C, 1))


def test_not_spd_info():
    """Z3: info = first failing global column (1-based)."""
    n, b = 8, 4
    A = np.asfortranarray(np.eye(n))
    A[5, 5] = -1.0
    F, info = _factor(A, b)
    assert info == 6


def test_pack_spec_example():
    """4x4 a_rc = 10r+c (1-based), b=2 -> tile(2,1) buffer [31,41,32,42]."""
    D = np.asfortranarray([[10.0 * r + c for c in range(1, 5)] for r in range(1, 5)])
    F = oracle.pack(D, 2)
    # tile (i=1, j=0) 0-based is at offset (1 + 0*2)*4
    assert list(F[4:8]) == [31.0, 41.0, 32.0, 42.0]
    assert np.array_equal(oracle.unpack(F, 4, 4, 2), D)


def test_host_pool_bitwise_equals_sequential():
    """The multicore baseline (oracle kernels on a host thread pool driven by the DAG,
    the paper's progress-table runtime) reproduces the sequential
    drivers bitwise for all three algorithms (SPEC.md:369 schedule independence)."""
    import oracle as o
    for alg, gen in (("chol", tilegen.spd), ("qr", tilegen.uniform), ("lu", tilegen.normal)):
        n, b, ib = 160, 32, 8
        A = gen(n, 9)
        F1, F2 = o.pack(A, b), o.pack(A, b)
        if alg == "chol":
            i1 = o.chol(F1, n, b)
            _, _, i2 = o.factor_par(alg, F2, n, b, ib, 6)
            assert i1 == i2 == 0
        elif alg == "qr":
            T1 = o.qr(F1, n, b, ib)
            T2, _, _ = o.factor_par(alg, F2, n, b, ib, 6)
            assert np.array_equal(T1, T2)
        else:
            L1, p1, i1 = o.lu(F1, n, b, ib)
            L2, p2, i2 = o.factor_par(alg, F2, n, b, ib, 6)
            assert np.array_equal(L1, L2) and np.array_equal(p1, p2) and i1 == i2
        assert np.array_equal(F1, F2), alg
    # Cholesky failure: same info as the sequential driver
    A = tilegen.spd(128, 1)
    A[70, 70] = -1e6
    F = o.pack(A, 32)
    assert o.factor_par("chol", F, 128, 32, 8, 4)[2] == o.chol(o.pack(A, 32), 128, 32)
