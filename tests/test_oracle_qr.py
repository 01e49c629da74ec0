"""Pins of the oracle's tiled QR (Algorithm 2; kernels PAPER.md:356-429,
inner blocking PAPER.md:637-653) against LAPACK (numpy 'raw' dgeqrf output), exact
permutation / triangular pins, the Hadamard closed form, explicit reflector products,
and the SPEC worked examples."""
import numpy as np
import pytest

import oracle
import tilegen


def _factor(A, b, ib):
    n = A.shape[0]
    F = oracle.pack(A, b)
    T = oracle.qr(F, n, b, ib)
    return F, T


def _explicit_T_check(V, tau, T, ib):
    """I - V T V^T must equal H_0 H_1 ... H_{ib-1} (the compact WY identity that
    defines T), computed here by explicit products."""
    m = V.shape[0]
    H = np.eye(m)
    for j in range(ib):
        v = V[:, j:j + 1]
        H = H @ (np.eye(m) - tau[j] * (v @ v.T))
    return np.max(np.abs(np.eye(m) - V @ T @ V.T - H))


@pytest.mark.parametrize("n,ib", [(32, 8), (24, 24), (40, 5)])
def test_single_tile_vs_lapack_raw(n, ib):
    """p = 1: V, tau and R elementwise equal to LAPACK dgeqrf (same dlarfg sign
    convention, Z6); T equals the dlarft factor of V via the explicit product."""
    A = tilegen.uniform(n, 3)
    F, T = _factor(A, n, ib)
    h, tau_ref = np.linalg.qr(A, mode="raw")
    Fref = h.T  # raw mode returns the Fortran array transposed
    assert np.max(np.abs(np.triu(F.reshape(n, n, order="F")) - np.triu(Fref))) <= 1e-14
    assert np.max(np.abs(np.tril(F.reshape(n, n, order="F"), -1) - np.tril(Fref, -1))) <= 1e-13
    Ts = T.reshape(ib, n, order="F")
    tau = np.concatenate([np.diag(Ts[:, s * ib:(s + 1) * ib]) for s in range(n // ib)])
    assert np.max(np.abs(tau - tau_ref)) <= 1e-14
    D = F.reshape(n, n, order="F")
    for s in range(n // ib):
        c0 = s * ib
        V = np.tril(D[c0:, c0:c0 + ib], -1)
        V[np.arange(ib), np.arange(ib)] = 1.0
        err = _explicit_T_check(V, tau[c0:c0 + ib], Ts[:, c0:c0 + ib], ib)
        assert err <= 1e-14
        assert np.array_equal(np.tril(Ts[:, c0:c0 + ib], -1), np.zeros((ib, ib)))


@pytest.mark.parametrize("n,b,ib", [(64, 16, 4), (96, 32, 8), (48, 16, 16), (60, 12, 3)])
def test_residual_orthogonality_vs_lapack(n, b, ib):
    A = tilegen.uniform(n, n + b)
    F, T = _factor(A, b, ib)
    R = oracle.qr_R(F, n, b)
    QR = oracle.qr_apply(F, T, R, n, b, ib, trans=False)
    assert np.linalg.norm(A - QR) / np.linalg.norm(A) <= 1e-14
    Q = oracle.qr_apply(F, T, np.eye(n), n, b, ib, trans=False)
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13 * n
    # Q^T applied to A gives R (the transposed apply path)
    QtA = oracle.qr_apply(F, T, A, n, b, ib, trans=True)
    assert np.max(np.abs(np.tril(QtA, -1))) <= 1e-13
    # R equal to LAPACK's up to row signs (Z16)
    Rref = np.linalg.qr(A, mode="r")
    sg = np.sign(np.diag(R)) * np.sign(np.diag(Rref))
    assert np.max(np.abs(R - sg[:, None] * Rref)) <= 1e-12


@pytest.mark.parametrize("n,b,ib", [(64, 16, 4), (32, 8, 8), (48, 12, 6)])
def test_permutation_pin_bitwise(n, b, ib):
    """Scaled permutation: every step exact; |R| = |D| diagonal, zero elsewhere."""
    A, d = tilegen.qr_perm(n, b)
    F, T = _factor(A, b, ib)
    R = oracle.qr_R(F, n, b)
    assert np.array_equal(np.abs(np.diag(R)), np.abs(d))
    assert np.array_equal(np.triu(R, 1), np.zeros((n, n)))
    Ts = T.reshape(-1)
    taus = []
    p = n // b
    for i in range(p):
        for k in range(p):
            S = T[(i + k * p) * ib * b:(i + k * p + 1) * ib * b].reshape(ib, b, order="F")
            for s in range(b // ib):
                taus.extend(np.diag(S[:, s * ib:(s + 1) * ib]))
    assert set(np.unique(taus)).issubset({0.0, 1.0})


@pytest.mark.parametrize("n,b,ib", [(32, 8, 4), (48, 16, 8)])
def test_upper_triangular_pin(n, b, ib):
    """Upper-triangular input: tau = 0 everywhere, R = A bitwise, V = 0, T = 0."""
    A = tilegen.qr_upper(n, 9)
    F, T = _factor(A, b, ib)
    D = oracle.unpack(F, n, n, b)
    assert np.array_equal(D, A)
    assert np.array_equal(T, np.zeros_like(T))


@pytest.mark.parametrize("n,b,ib", [(64, 16, 4), (128, 32, 8)])
def test_hadamard_closed_form(n, b, ib):
    """H^T H = n I  =>  |R| = sqrt(n) I (SURVEY C5 closed form)."""
    A = tilegen.hadamard(n)
    F, T = _factor(A, b, ib)
    R = oracle.qr_R(F, n, b)
    assert np.max(np.abs(np.abs(np.diag(R)) - np.sqrt(n))) <= 1e-13 * np.sqrt(n)
    assert np.max(np.abs(np.triu(R, 1))) <= 1e-13 * np.sqrt(n)


def test_ib_independence():
    """R and V are mathematically independent of ib (C5)."""
    n, b = 64, 16
    A = tilegen.uniform(n, 21)
    F1, _ = _factor(A, b, 4)
    F2, _ = _factor(A, b, 16)
    assert np.max(np.abs(F1 - F2)) <= 1e-13


def test_spec_examples():
    b = 4
    # geqrt(I) -> R = I, T = 0
    A = np.asfortranarray(np.eye(b))
    T = oracle.geqrt(A, 2)
    assert np.array_equal(A, np.eye(b)) and np.array_equal(T, np.zeros_like(T))
    # tsqrt with zero A -> R unchanged, V = 0, T = 0
    R = np.asfortranarray(np.triu(np.arange(1.0, 17.0).reshape(4, 4)))
    R0 = R.copy()
    Z = np.zeros((b, b), order="F")
    T = oracle.tsqrt(R, Z, 2)
    assert np.array_equal(R, R0) and not Z.any() and not T.any()
    # b=2, s=2, R=I, A=I -> |new R diag| = sqrt(2)
    R = np.asfortranarray(np.eye(2))
    A = np.asfortranarray(np.eye(2))
    oracle.tsqrt(R, A, 2)
    assert np.allclose(np.abs(np.diag(R)), np.sqrt(2.0), atol=1e-15, rtol=0)


def test_ssrfb_reproduces_tsqrt_R():
    """applying SSRFB to the columns TSQRT factored reproduces its R."""
    b, ib = 8, 4
    r = np.random.default_rng(1)
    R = np.asfortranarray(np.triu(r.standard_normal((b, b))))
    A = np.asfortranarray(r.standard_normal((b, b)))
    R2, A2 = R.copy(order="F"), A.copy(order="F")
    T = oracle.tsqrt(R, A, ib)
    oracle.ssrfb(A, T, R2, A2, ib)
    assert np.max(np.abs(np.triu(R2) - np.triu(R))) <= 1e-13
    assert np.max(np.abs(A2)) <= 1e-13


def test_larfb_matches_dense_product():
    """LARFB equals the explicit Q^T product built from the reflectors."""
    b, ib = 12, 4
    r = np.random.default_rng(2)
    A = np.asfortranarray(r.standard_normal((b, b)))
    h, tau = np.linalg.qr(A.copy(), mode="raw")
    F = A.copy(order="F")
    T = oracle.geqrt(F, ib)
    C = np.asfortranarray(r.standard_normal((b, b)))
    C2 = C.copy(order="F")
    oracle.larfb(F, T, C2, ib)
    V = np.tril(F, -1) + np.eye(b)
    Q = np.eye(b)
    for j in range(b):
        v = V[:, j:j + 1]
        Q = Q @ (np.eye(b) - tau[j] * v @ v.T)
    assert np.max(np.abs(C2 - Q.T @ C)) <= 1e-13
