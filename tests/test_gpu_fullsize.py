"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(one persistent launch per factorization, one CTA per SM).

* configs 2 and 3 (n = 4096): element-wise against the oracle run on the same input
  (per-tile tolerances of DESIGN.md §3; LU pivots bit-identical) — the oracle takes about a
  minute of host time here.
* configs 4 and 5 (n = 32768): the oracle cannot factor them in test time, so the
  north_star invariants are estimated with k Gaussian probe vectors X (E||E X||_F^2 =
  k ||E||_F^2): ||A - L L^T||_F / ||A||_F <= 1e-13, ||A - Q R||_F / ||A||_F <= 1e-13 and
  ||Q^T Q - I||_F <= 1e-13 n, with Q applied by the oracle's compact-WY routine.
"""
import numpy as np
import pytest

import oracle
import tilegen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from _gpu_util import gpu_factor, lu_certified, lu_tile_tolerances, oracle_factor, rel, strip, tile_errors  # noqa: E402
from paper_0709_1272_b200 import tilefact as tf  # noqa: E402

TOL = 1e-10


def test_config2_qr_full_parity():
    n, b, ib = 4096, 256, 32
    A = tilegen.uniform(n, 0)
    G, GT, _, _ = gpu_factor("qr", A, b, ib)
    O, OT, _, _ = oracle_factor("qr", A, b, ib)
    errs = tile_errors("qr", G, O, n, b)
    assert max(errs.values()) <= TOL, max(errs.items(), key=lambda kv: kv[1])
    p = n // b
    worst = max(rel(strip(GT, p, b, ib, i, k), strip(OT, p, b, ib, i, k)) for k in range(p) for i in range(k, p))
    assert worst <= TOL


def test_config3_lu_full_parity():
    """Config 3 at full size: pivots bit-exact, per-tile U/L and the L strips within the
    C5 tolerance (the perturbed oracle run must keep the same pivots, pivot margin
    reported), and BASELINE's LU residual ||A - N U||_F / ||A||_F <= max(1e-12, 2x the
    oracle's own value) (reading Z14)."""
    n, b, ib = 4096, 256, 32
    c = lu_certified(n, b, ib, 0)
    A, O, OL, Op = c["A"], c["O"], c["OL"], c["Op"]
    G, GL, Gp, gi = gpu_factor("lu", A, b, ib)
    assert gi == c["info"] == 0
    p = n // b
    for k in range(p):
        for i in range(k, p):
            o = (i + k * p) * b
            assert np.array_equal(Gp[o:o + b], Op[o:o + b]), (i, k)
    tol, sig = lu_tile_tolerances(c, n, b)
    errs = tile_errors("lu", G, O, n, b)
    for key, e in errs.items():
        assert e <= tol[key], (key, e, sig[key])
    for k in range(p):
        for i in range(k + 1, p):
            assert rel(strip(GL, p, b, ib, i, k), strip(OL, p, b, ib, i, k)) <= tol[(i, k)], (i, k)
    nA = np.linalg.norm(A)
    rg = np.linalg.norm(A - oracle.lu_apply_N(G, GL, Gp, oracle.lu_U(G, n, b), n, b, ib)) / nA
    ro = np.linalg.norm(A - oracle.lu_apply_N(O, OL, Op, oracle.lu_U(O, n, b), n, b, ib)) / nA
    print(f"[config 3] ||A - NU||/||A||: gpu {rg:.3e} oracle {ro:.3e}; margin {c['margin']:.3g}")
    assert rg <= max(1e-12, 2 * ro), (rg, ro)


def _device_matrix(gen, n, seed):
    if gen == "spd":
        return tilegen.spd_torch(n, seed, torch.device("cuda"))
    return tilegen.uniform_torch(n, seed, -0.5, 0.5, torch.device("cuda"))


def test_config4_chol_full_residual():
    n, b, ib = 32768, 512, 64
    dense = _device_matrix("spd", n, 0)          # row-major buffer; its column-major reading is A (symmetric)
    T = torch.empty(n * n, dtype=torch.float64, device="cuda")
    tf.tile_pack(n, n, b, dense.view(-1), T)
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    tf.tile_chol(n, b, ib, T, info)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    D = torch.empty(n * n, dtype=torch.float64, device="cuda")
    tf.tile_unpack(n, n, b, T, D)
    del T
    L = torch.tril(D.view(n, n).t())
    del D
    A = dense.t()
    g = torch.Generator(device="cuda").manual_seed(3)
    X = torch.randn(n, 8, dtype=torch.float64, device="cuda", generator=g)
    R = A @ X - L @ (L.t() @ X)
    # E[||E X||_F^2] = k ||E||_F^2 for X with k i.i.d. N(0,1) columns: ||E X||_F / sqrt(k)
    # estimates ||A - L L^T||_F, held to north_star's 1e-13 relative bound
    k = X.shape[1]
    res = float(torch.linalg.norm(R) / (k ** 0.5 * torch.linalg.norm(A)))
    print(f"[config 4] est ||A - LL^T||_F/||A||_F = {res:.3e}")
    assert res <= 1e-13, res
    # lower-triangular with a positive diagonal
    assert bool((torch.diagonal(L) > 0).all())


def test_config5_qr_full_residual_and_orthogonality():
    n, b, ib = 32768, 512, 64
    dense = _device_matrix("uniform", n, 0)      # row-major buffer = A^T; A is its column-major reading
    T = torch.empty(n * n, dtype=torch.float64, device="cuda")
    tf.tile_pack(n, n, b, dense.view(-1), T)
    Tq = torch.zeros(tf.tile_qr_t_elems(n, b, ib), dtype=torch.float64, device="cuda")
    tf.tile_qr(n, b, ib, T, Tq)
    torch.cuda.synchronize()
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.randn(n, 4, dtype=torch.float64, device="cuda", generator=g)
    AX = (dense.t() @ X).cpu().numpy()
    nA = float(torch.linalg.norm(dense))
    del dense
    D = torch.empty(n * n, dtype=torch.float64, device="cuda")
    tf.tile_unpack(n, n, b, T, D)
    RX = (torch.triu(D.view(n, n).t()) @ X).cpu().numpy()
    del D
    G = T.cpu().numpy()
    GT = Tq.cpu().numpy()
    del T, Tq
    torch.cuda.empty_cache()
    QRX = oracle.qr_apply(G, GT, RX, n, b, ib)
    k = X.shape[1]
    # ||E X||_F / sqrt(k) estimates ||A - QR||_F (probe estimator)
    res = np.linalg.norm(AX - QRX) / (k ** 0.5 * nA)
    Y = np.asfortranarray(np.random.default_rng(6).standard_normal((n, 3)))
    QY = oracle.qr_apply(G, GT, Y, n, b, ib)
    back = oracle.qr_apply(G, GT, QY, n, b, ib, trans=True)
    # ||(Q^T Q - I) Y||_F / sqrt(3) estimates ||Q^T Q - I||_F, bound 1e-13 n (north_star)
    orth = np.linalg.norm(back - Y) / 3 ** 0.5
    print(f"[config 5] est ||A - QR||_F/||A||_F = {res:.3e}, est ||Q^T Q - I||_F = {orth:.3e}")
    assert res <= 1e-13, res
    assert orth <= 1e-13 * n, orth


def test_config6_lu_full_residual_and_solve():
    """NEXT-1 (Alg. 3 at n = 32768, b = 512, ib = 64, the launch bench.py --config 6 times):
    the oracle cannot factor it in test time, so properties that hold at any size are checked:
    every stored multiplier |l| <= 1 (GETWP's pivots always eliminate with the
    larger element), ||A - N U||_F / ||A||_F estimated with Gaussian probes (N applied with
    the GPU's tile_lu_apply_N, itself parity-tested against the oracle), and the backward
    error of a solve with tile_getrs."""
    n, b, ib = 32768, 512, 64
    dense = tilegen.normal_torch(n, 0, torch.device("cuda"))   # row-major buffer = A^T
    T = torch.empty(n * n, dtype=torch.float64, device="cuda")
    tf.tile_pack(n, n, b, dense.view(-1), T)
    Ls = torch.zeros(tf.tile_lu_l_elems(n, b, ib), dtype=torch.float64, device="cuda")
    piv = torch.zeros(tf.tile_lu_ipiv_elems(n, b), dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    tf.tile_lu(n, b, ib, T, Ls, piv, info)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    D = torch.empty(n * n, dtype=torch.float64, device="cuda")
    tf.tile_unpack(n, n, b, T, D)
    F = D.view(n, n).t()                                       # the factored matrix, (row, col)
    assert float(torch.tril(F, -1).abs().max()) <= 1.0
    assert float(Ls.abs().max()) <= 1.0
    U = torch.triu(F)
    del D
    A = dense.t()
    g = torch.Generator(device="cuda").manual_seed(11)
    X = torch.randn(n, 4, dtype=torch.float64, device="cuda", generator=g)
    Y = (U @ X).t().contiguous()                               # (4, n) = column-major n x 4
    tf.tile_lu_apply_N(n, b, ib, T, Ls, piv, Y)
    E = A @ X - Y.t()
    res = float(torch.linalg.norm(E) / (2.0 * torch.linalg.norm(A)))
    print(f"[config 6] est ||A - NU||_F/||A||_F = {res:.3e}")
    # GETWP's factorization error grows with p and n (the lab: 1.5e-14 at p = 1 to 1.2e-12 at
    # p = 128 for n = 2048; test_config6_method_level pins GPU = oracle level at p = 16 with
    # this tile shape); no oracle value exists at n = 32768, so this is a sanity bound that a
    # wrong elimination (O(1) errors) cannot pass, and the strong check is the solve below
    assert res <= 1e-8, res
    y = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    x = y.clone()
    tf.tile_getrs(n, b, ib, T, Ls, piv, x)
    be = float((y - A @ x).abs().max() / (torch.linalg.matrix_norm(A, ord=float("inf")) * x.abs().max()))
    print(f"[config 6] solve backward error = {be:.3e}")
    assert be <= 1e-12, be


def test_config6_method_level_p16():
    """The b = 512 / ib = 64 LU path at p = 16 (n = 8192): the GPU's ||A - N U||_F / ||A||_F
    is at the oracle's own level (<= max(1e-12, 2x the oracle's), BASELINE's LU residual
    reading Z14); the oracle runs on all host cores (its thread-pool executor, bitwise equal
    to the sequential driver).  Pivots are NOT required to agree here: at this depth the
    oracle's own rounding spread exceeds some pivot gaps (seed 3: first disagreement at tile
    (14,12) column 337, winner / runner-up |x| 6.0839512 / 6.0839224, relative gap 4.7e-6,
    C5 pivot margin 0.24 — a pivot-fragile seed under reading C5, diagnosed with
    tools/lu_pivot_diag.py); both factorizations are valid GETWP runs, and the bit-exact
    pivot requirement is carried by the certified seeds of test_gpu_parity / config 3."""
    n, b, ib = 8192, 512, 64
    A = tilegen.normal(n, 3)
    G, GL, Gp, gi = gpu_factor("lu", A, b, ib)
    import os
    F = oracle.pack(A, b)
    OL, Op, oi = oracle.factor_par("lu", F, n, b, ib, len(os.sched_getaffinity(0)))
    assert gi == oi == 0
    p = n // b
    same = sum(np.array_equal(Gp[(i + k * p) * b:(i + k * p + 1) * b], Op[(i + k * p) * b:(i + k * p + 1) * b])
               for k in range(p) for i in range(k, p))
    print(f"[n=8192 b=512 ib=64] identical pivot vectors: {same} of {p * (p + 1) // 2}")
    # ||A - N U||_F estimated with the same 8 Gaussian probes for both (E||EX||^2 = k||E||^2)
    X = np.asfortranarray(np.random.default_rng(8).standard_normal((n, 8)))
    AX, nA = A @ X, np.linalg.norm(A) * 8 ** 0.5
    rg = np.linalg.norm(AX - oracle.lu_apply_N(G, GL, Gp, oracle.lu_U(G, n, b) @ X, n, b, ib)) / nA
    ro = np.linalg.norm(AX - oracle.lu_apply_N(F, OL, Op, oracle.lu_U(F, n, b) @ X, n, b, ib)) / nA
    print(f"[n=8192 b=512 ib=64] est ||A - NU||_F/||A||_F: gpu {rg:.3e} oracle {ro:.3e}")
    assert rg <= max(1e-12, 2 * ro), (rg, ro)
