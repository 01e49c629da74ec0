"""Pins of the oracle's tiled LU with incremental pivoting (Algorithm 3, PAPER.md:560-576;
kernels PAPER.md:476-533; L-strip footnote PAPER.md:542-544) against LAPACK (scipy
getrf: b = n => GEPP), brute-force GEWP (b = 1), the exact
dyadic pin, the N U = A identity (Eq. eq:GETWPcompact), the multiplier
bound and the SPEC worked examples."""
import numpy as np
import pytest
import scipy.linalg

import oracle
import tilegen


def _factor(A, b, ib):
    n = A.shape[0]
    F = oracle.pack(A, b)
    Ls, piv, info = oracle.lu(F, n, b, ib)
    return F, Ls, piv, info


def _rel_resid(A, F, Ls, piv, n, b, ib):
    U = oracle.lu_U(F, n, b)
    NU = oracle.lu_apply_N(F, Ls, piv, U, n, b, ib)
    return np.linalg.norm(A - NU) / np.linalg.norm(A)


@pytest.mark.parametrize("n,ib", [(32, 8), (40, 40), (48, 6)])
def test_b_equals_n_is_gepp(n, ib):
    """b = n: GETWP reduces to GEPP; pivots identical to LAPACK dgetrf,
    L and U elementwise to rounding."""
    A = tilegen.normal(n, n)
    F, Ls, piv, info = _factor(A, n, ib)
    lu_ref, piv_ref = scipy.linalg.lu_factor(A)
    assert info == 0
    assert np.array_equal(piv[:n], piv_ref.astype(np.int32) + 1)
    D = F.reshape(n, n, order="F")
    assert np.max(np.abs(D - lu_ref)) <= 1e-13 * max(1.0, np.abs(lu_ref).max())
    # brute-force unblocked GEPP: same pivots, same factors to rounding
    Dg, pg, ig = oracle.ref_gepp(A)
    assert np.array_equal(pg, piv[:n]) and ig == 0
    assert np.max(np.abs(Dg - D)) <= 1e-13 * max(1.0, np.abs(D).max())


def test_gepp_ref_vs_lapack():
    A = tilegen.normal(30, 4)
    Dg, pg, _ = oracle.ref_gepp(A)
    lu_ref, piv_ref = scipy.linalg.lu_factor(A)
    assert np.array_equal(pg, piv_ref.astype(np.int32) + 1)
    assert np.max(np.abs(Dg - lu_ref)) <= 1e-13


@pytest.mark.parametrize("n", [8, 17, 24])
def test_b1_is_gewp_bitwise(n):
    """b = 1: GETWP reduces to GEWP.  Same operations in the same order,
    so U, multipliers and swap decisions match the brute-force GEWP bitwise."""
    A = tilegen.normal(n, 100 + n)
    F, Ls, piv, info = _factor(A, 1, 1)
    Dw, sw, infow = oracle.ref_gewp(A)
    D = F.reshape(n, n, order="F")  # b = 1: BDL == column-major
    assert np.array_equal(D, Dw)
    # tile (i,k) pivot: 2 (= b+0+1) when the bottom row won, else 1
    P = piv.reshape(n, n, order="F")
    for k in range(n):
        for i in range(k + 1, n):
            assert P[i, k] == (2 if sw[k, i] else 1)


@pytest.mark.parametrize("n,b,ib,seed", [(64, 16, 4, 0), (96, 32, 8, 1), (48, 48, 12, 2), (64, 8, 8, 3)])
def test_exact_dyadic_pin(n, b, ib, seed):
    """A = L0 U0 (dyadic, |L0| <= 3/4): no swap anywhere, U = U0 and multipliers = L0
    bitwise, Ls strips stay zero, and N U0 = A exactly (N = L0)."""
    A, L0, U0 = tilegen.lu_exact(n, seed)
    F, Ls, piv, info = _factor(A, b, ib)
    assert info == 0
    p = n // b
    P = piv.reshape(p * p, b)
    for i in range(p):
        for k in range(i + 1):
            v = P[i + k * p]
            assert np.array_equal(v, np.arange(1, b + 1)), (i, k)
    D = oracle.unpack(F, n, n, b)
    assert np.array_equal(np.triu(D), U0)
    assert np.array_equal(np.tril(D, -1), np.tril(L0, -1))
    assert not Ls.any()
    NU = oracle.lu_apply_N(F, Ls, piv, U0, n, b, ib)
    assert np.array_equal(NU, A)


@pytest.mark.parametrize("n,b,ib", [(128, 32, 8), (96, 16, 4), (64, 64, 16), (120, 24, 6)])
def test_factorization_residual_and_multipliers(n, b, ib):
    """||A - N U||_F/||A||_F small (C4, Z14) and every multiplier |l| <= 1."""
    A = tilegen.normal(n, 7 * n + b)
    F, Ls, piv, info = _factor(A, b, ib)
    assert info == 0
    assert _rel_resid(A, F, Ls, piv, n, b, ib) <= 1e-13
    D = oracle.unpack(F, n, n, b)
    assert np.abs(np.tril(D, -1)).max() <= 1.0
    assert np.abs(Ls).max() <= 1.0
    # pivot ranges (Z13)
    p = n // b
    P = piv.reshape(p * p, b)
    for k in range(p):
        assert P[k + k * p].min() >= 1 and P[k + k * p].max() <= b
        for i in range(k + 1, p):
            assert P[i + k * p].min() >= 1 and P[i + k * p].max() <= 2 * b


def test_ib_independence():
    """Pivots and U are mathematically independent of ib (C5)."""
    n, b = 96, 32
    A = tilegen.normal(n, 5)
    F1, Ls1, p1, _ = _factor(A, b, 4)
    F2, Ls2, p2, _ = _factor(A, b, 32)
    assert np.array_equal(p1, p2)
    U1, U2 = oracle.lu_U(F1, n, b), oracle.lu_U(F2, n, b)
    assert np.max(np.abs(U1 - U2)) <= 1e-12 * np.abs(U1).max()
    assert _rel_resid(A, F2, Ls2, p2, n, b, 32) <= 1e-13


def test_spec_getrf_swap():
    """[[0,1],[1,0]] -> P swaps rows, L = I, U = I."""
    A = np.asfortranarray([[0.0, 1.0], [1.0, 0.0]])
    piv, info = oracle.getrf(A, 2)
    assert list(piv) == [2, 2] and info == 0
    assert np.array_equal(A, np.eye(2))


def test_spec_tstrf_b1():
    """b=1, u=[1], a=[3] -> P=[2], U=[3], multiplier 1/3."""
    U = np.asfortranarray([[1.0]])
    A = np.asfortranarray([[3.0]])
    Ls, piv, info = oracle.tstrf(U, A, 1)
    assert list(piv) == [2] and U[0, 0] == 3.0 and A[0, 0] == 1.0 / 3.0 and info == 0


def test_spec_ssssm_single_swap():
    """single swap, L = I (zero multipliers) -> rows exchanged."""
    b = 2
    L = np.zeros((b, b), order="F")
    Ls = np.zeros((b, b), order="F")
    piv = np.array([3, 2], dtype=np.int32)  # top row 0 <-> bottom row 0
    U = np.asfortranarray([[1.0, 2.0], [0.0, 3.0]])
    A = np.asfortranarray([[5.0, 6.0], [7.0, 8.0]])
    oracle.ssssm(L, Ls, piv, U, A, b)
    assert np.array_equal(U, [[5.0, 6.0], [0.0, 3.0]])
    assert np.array_equal(A, [[1.0, 2.0], [7.0, 8.0]])


def test_gessm_one_elimination():
    """P = id, l21 = 2 -> row2 := row2 - 2 row1."""
    L = np.asfortranarray([[1.0, 0.0], [2.0, 1.0]])
    piv = np.array([1, 2], dtype=np.int32)
    A = np.asfortranarray([[1.0, 1.0], [0.0, 1.0]])
    oracle.gessm(L, piv, A, 2)
    assert np.array_equal(A, [[1.0, 1.0], [-2.0, -1.0]])


def test_zero_pivot_info():
    """Z3: exactly singular column -> info = first zero-pivot global column."""
    n, b = 8, 4
    A = np.asfortranarray(np.eye(n))
    A[:, 5] = 0.0
    F, Ls, piv, info = _factor(A, b, 2)
    assert info == 6


def test_flop_formulas():
    """SSRFB 4b^3 + s b^2, SSSSM 2b^3 + s b^2; the sum over the
    tiled QR tasks approaches 4n^3/3 (1 + s/4b) (Z7)."""
    b, s = 200, 40
    assert oracle.kernel_flops("ssrfb", b, s) == 4 * b**3 + s * b**2
    assert oracle.kernel_flops("ssssm", b, s) == 2 * b**3 + s * b**2
    p = 400
    n = p * b
    tot = sum(oracle.kernel_flops("ssrfb", b, s) * (p - k) ** 2 for k in range(1, p + 1))
    assert abs(tot / (4 * n**3 / 3 * (1 + s / (4 * b))) - 1) < 0.01
    tot = sum(oracle.kernel_flops("ssssm", b, s) * (p - k) ** 2 for k in range(1, p + 1))
    assert abs(tot / (2 * n**3 / 3 * (1 + s / (2 * b))) - 1) < 0.01
    # kinds without a printed count in the paper are not provided
    assert np.isnan(oracle.kernel_flops("gemm", b, s)) and np.isnan(oracle.kernel_flops("larfb", b, s))
    # s = b gives the paper's 25% overhead
    assert (1 + b / (4 * b)) == 1.25


def test_decision_recorder_pins():
    """C5 instrumentation: the recorder does not change the arithmetic, records one
    decision per pivot (p(p+1)/2 * b), and for p = 1 (GEPP) the first
    decision is (max |A[:,0]|, second-largest |A[:,0]|) of the input, by brute force."""
    n, b, ib = 96, 32, 8
    A = tilegen.normal(n, 4)
    F = oracle.pack(A, b)
    Ls0, piv0, info0 = oracle.lu(F.copy(), n, b, ib)
    Ls1, piv1, info1, dec = oracle.lu_decisions(F.copy(), n, b, ib)
    assert np.array_equal(Ls0, Ls1) and np.array_equal(piv0, piv1) and info0 == info1 == 0
    p = n // b
    assert dec.shape == (p * (p + 1) // 2 * b, 2)
    assert (dec[:, 0] >= dec[:, 1]).all()
    A1 = tilegen.normal(32, 5)
    _, _, _, d1 = oracle.lu_decisions(oracle.pack(A1, 32), 32, 32, 8)
    col = np.sort(np.abs(A1[:, 0]))
    assert d1[0, 0] == col[-1] and d1[0, 1] == col[-2]
    # the unperturbed run against itself has an infinite-like margin; a perturbed run
    # with the same pivots has a finite one
    assert oracle.pivot_margin(dec, dec) >= 2.0 ** 40
