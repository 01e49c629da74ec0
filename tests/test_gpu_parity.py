"""GPU parity: the CUDA path (through the C-ABI) vs the oracle on the same seeded inputs.

Sizes span several tiles, ragged work-item tails (b not a multiple of the 128-row /
64-column item sizes), odd b (8-byte copy path), p = 1, and both panel paths (panel in
shared memory vs in global memory when b*ib is too large).  Tolerances: DESIGN.md §3.
"""
import numpy as np
import pytest

import oracle
import tilegen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from _gpu_util import (gpu_factor, gpu_pack, lu_certified, lu_tile_tolerances, oracle_factor,  # noqa: E402
                       rel, strip, tile, tile_errors)
from paper_0709_1272_b200 import tilefact as tf  # noqa: E402

TOL = 1e-10


# ------------------------------------------------------------------ layout

@pytest.mark.parametrize("m,n,b", [(8, 8, 2), (96, 64, 32), (63, 42, 21), (256, 256, 128)])
def test_pack_unpack_bitwise(m, n, b):
    A = tilegen.uniform(n, 1, m=m)
    T = gpu_pack(A, b)
    assert np.array_equal(T.cpu().numpy(), oracle.pack(A, b))
    D = torch.empty(m * n, dtype=torch.float64, device="cuda")
    tf.tile_unpack(m, n, b, T, D)
    assert np.array_equal(D.cpu().numpy().reshape(n, m).T, A)


# ------------------------------------------------------------------ Cholesky

@pytest.mark.parametrize("n,b,ib,seed", [
    (1024, 128, 32, 0),   # config 1 (BASELINE configs[0])
    (384, 96, 32, 1),     # ragged 128-row items
    (200, 40, 8, 2),
    (63, 21, 7, 3),       # odd b: 8-byte copy path
    (64, 64, 16, 4),      # p = 1
    (16, 1, 1, 5),        # b = 1
    (640, 160, 32, 6),
    (1536, 512, 64, 7),   # config-4 tile shape, p = 3: blocked POTRF, GEMM strips
    (1024, 256, 32, 8),
    (768, 384, 32, 9),    # b = 384: blocked POTRF over three 128-column panels
])
def test_chol_parity(n, b, ib, seed):
    A = tilegen.spd(n, seed)
    G, _, _, gi = gpu_factor("chol", A, b, ib)
    O, _, _, oi = oracle_factor("chol", A, b, ib)
    assert gi == 0 and oi == 0
    errs = tile_errors("chol", G, O, n, b)
    assert max(errs.values()) <= TOL, max(errs.items(), key=lambda kv: kv[1])
    # upper tiles and strict upper triangle of diagonal tiles untouched (Z2)
    p = n // b
    A0 = oracle.pack(A, b)
    for j in range(p):
        for i in range(p):
            if i < j:
                assert np.array_equal(tile(G, p, b, i, j), tile(A0, p, b, i, j))
            elif i == j:
                assert np.array_equal(np.triu(tile(G, p, b, i, i), 1), np.triu(tile(A0, p, b, i, i), 1))
    L = oracle.tile_lower_L(G, n, b)
    assert np.linalg.norm(A - L @ L.T) / np.linalg.norm(A) <= 1e-13


@pytest.mark.parametrize("n,b", [(256, 64), (384, 128), (90, 30),
                                 (768, 256), (1024, 512), (768, 384)])  # blocked POTRF, 4-sub-tile GEMM strips
def test_chol_exact_pin_bitwise(n, b):
    A, L0 = tilegen.chol_exact(n, n + b)
    G, _, _, gi = gpu_factor("chol", A, b, b // 2)
    assert gi == 0
    assert np.array_equal(oracle.tile_lower_L(G, n, b), L0)


def test_chol_not_spd_info():
    n, b = 256, 64
    A = tilegen.spd(n, 3)
    A[150, 150] = -1e6
    G, _, _, gi = gpu_factor("chol", A, b, 16)
    O, _, _, oi = oracle_factor("chol", A, b, 16)
    assert gi == oi and gi > 0


# ------------------------------------------------------------------ QR

@pytest.mark.parametrize("n,b,ib,seed", [
    (768, 256, 32, 0),    # config-2 tile shape, p = 3
    (512, 128, 16, 1),
    (480, 96, 24, 2),     # ragged 64-column slabs
    (90, 30, 5, 3),       # odd ib
    (512, 512, 64, 4),    # p = 1, panel in global memory (b*ib too large for smem)
    (63, 21, 7, 5),       # odd b
    (1024, 512, 64, 6),   # config-5 tile shape, p = 2 (T12 coupling, ib = 64)
    (640, 128, 32, 7),    # b = 128 slab path, p = 5
    (1536, 512, 64, 8),   # config-5 tile shape, p = 3: chained TSQRT / SSRFB with i > k + 1
    (768, 384, 32, 9),    # b = 384: reference-blocked kernels (not a register-slab size)
])
def test_qr_parity(n, b, ib, seed):
    A = tilegen.uniform(n, seed)
    G, GT, _, _ = gpu_factor("qr", A, b, ib)
    O, OT, _, _ = oracle_factor("qr", A, b, ib)
    errs = tile_errors("qr", G, O, n, b)
    assert max(errs.values()) <= TOL, max(errs.items(), key=lambda kv: kv[1])
    p = n // b
    for k in range(p):
        for i in range(k, p):
            assert rel(strip(GT, p, b, ib, i, k), strip(OT, p, b, ib, i, k)) <= TOL, (i, k)
    # invariants on the GPU factors, applied through the oracle's Q
    R = oracle.qr_R(G, n, b)
    QR = oracle.qr_apply(G, GT, R, n, b, ib)
    assert np.linalg.norm(A - QR) / np.linalg.norm(A) <= 1e-13


@pytest.mark.parametrize("n,b,ib", [(256, 64, 16), (96, 32, 8),
                                    (384, 128, 32), (512, 256, 32), (512, 512, 64)])  # register-slab sizes
def test_qr_exact_pins(n, b, ib):
    A, d = tilegen.qr_perm(n, 11)
    G, GT, _, _ = gpu_factor("qr", A, b, ib)
    R = oracle.qr_R(G, n, b)
    assert np.array_equal(np.abs(np.diag(R)), np.abs(d))
    assert not np.triu(R, 1).any()
    O, OT, _, _ = oracle_factor("qr", A, b, ib)
    assert np.array_equal(G, O) and np.array_equal(GT, OT)
    U = tilegen.qr_upper(n, 5)
    G, GT, _, _ = gpu_factor("qr", U, b, ib)
    assert np.array_equal(oracle.unpack(G, n, n, b), U)
    assert not GT.any()


# ------------------------------------------------------------------ LU

@pytest.mark.parametrize("n,b,ib,seed", [
    (768, 256, 32, 0),    # config-3 tile shape, p = 3
    (512, 128, 16, 1),
    (480, 96, 24, 2),
    (90, 30, 5, 3),
    (512, 512, 64, 4),    # p = 1 (= GEPP), panel in global memory
    (63, 21, 7, 5),
    (1024, 512, 32, 6),   # b = 512 slab panels, p = 2
    (640, 128, 32, 7),    # b = 128 slab path, p = 5
    (1024, 512, 64, 8),   # ib = 64 register block solves (GESSM / SSSSM), p = 2
    (1536, 512, 64, 9),   # NEXT-1 tile shape, p = 3: chained TSTRF / SSSSM with i > k + 1
    (768, 384, 32, 10),   # b = 384: reference-blocked kernels (not a register-slab size)
    (768, 256, 64, 11),   # ib = 64 slab GETRF / TSTRF (two slabs per inner block), b = 256
    (512, 128, 64, 12),   # ib = 64, b = 128
])
def test_lu_parity(n, b, ib, seed):
    c = lu_certified(n, b, ib, seed)
    A, O, OL, Op = c["A"], c["O"], c["OL"], c["Op"]
    G, GL, Gp, gi = gpu_factor("lu", A, b, ib)
    assert gi == 0 and c["info"] == 0
    p = n // b
    # pivots bit-exact on the stored vectors (k,k) and (i>k,k)
    for k in range(p):
        for i in range(k, p):
            o = (i + k * p) * b
            assert np.array_equal(Gp[o:o + b], Op[o:o + b]), (i, k)
    errs = tile_errors("lu", G, O, n, b)
    tol, sig = lu_tile_tolerances(c, n, b)
    for key, e in errs.items():
        assert e <= tol[key], (key, e, sig[key])
    for k in range(p):
        for i in range(k + 1, p):
            assert rel(strip(GL, p, b, ib, i, k), strip(OL, p, b, ib, i, k)) <= tol[(i, k)]
    U = oracle.lu_U(G, n, b)
    NU = oracle.lu_apply_N(G, GL, Gp, U, n, b, ib)
    ro = np.linalg.norm(A - oracle.lu_apply_N(O, OL, Op, oracle.lu_U(O, n, b), n, b, ib)) / np.linalg.norm(A)
    assert np.linalg.norm(A - NU) / np.linalg.norm(A) <= max(1e-12, 2 * ro)


@pytest.mark.parametrize("n,b,ib", [(256, 64, 16), (96, 32, 8), (128, 128, 32),
                                    (384, 128, 32), (512, 256, 32), (512, 512, 64),  # register-slab sizes
                                    (768, 256, 64), (1024, 512, 64)])  # ib = 64 slab GETRF / TSTRF
def test_lu_exact_pin_bitwise(n, b, ib):
    A, L0, U0 = tilegen.lu_exact(n, 3)
    G, GL, Gp, gi = gpu_factor("lu", A, b, ib)
    O, OL, Op, oi = oracle_factor("lu", A, b, ib)
    assert gi == 0
    assert np.array_equal(G, O) and np.array_equal(Gp, Op) and np.array_equal(GL, OL)
    assert np.array_equal(np.triu(oracle.unpack(G, n, n, b)), U0)


def test_lu_b1_is_gewp():
    n = 24
    A = tilegen.normal(n, 9)
    G, GL, Gp, gi = gpu_factor("lu", A, 1, 1)
    Dw, sw, _ = oracle.ref_gewp(A)
    assert np.max(np.abs(G.reshape(n, n).T - Dw)) <= 1e-12
    P = Gp.reshape(n, n).T
    for k in range(n):
        for i in range(k + 1, n):
            assert P[i, k] == (2 if sw[k, i] else 1)


@pytest.mark.parametrize("n,b,ib,col", [
    (128, 32, 8, 70),      # reference-blocked kernels
    (512, 128, 32, 70),    # register-slab GETRF / TSTRF, zero pivot in the third slab
    (768, 256, 32, 296),   # zero column b + 40: second tile column, second slab
])
def test_lu_singular_info(n, b, ib, col):
    A = tilegen.normal(n, 2)
    A[:, col] = 0.0
    _, _, _, gi = gpu_factor("lu", A, b, ib)
    _, _, _, oi = oracle_factor("lu", A, b, ib)
    assert gi == oi == col + 1


# ------------------------------------------------------------------ end-to-end host path

@pytest.mark.parametrize("alg,n,b,ib", [("chol", 1024, 128, 32), ("qr", 1024, 256, 32), ("lu", 1024, 256, 32),
                                        ("chol", 1536, 512, 64)])
def test_factor_host_overlapped_equals_device(alg, n, b, ib):
    """tile_factor_host streams tile columns in / out while the factorization runs
    (ARRIVE / DONE tasks in the DAG); the factors are bitwise those of the device call."""
    A = {"chol": tilegen.spd, "qr": tilegen.uniform, "lu": tilegen.normal}[alg](n, 13)
    G, GA, GP, gi = gpu_factor(alg, A, b, ib)
    hA = gpu_pack(A, b).cpu().pin_memory()
    if alg == "chol":
        # upper tiles are neither read nor written: start them at NaN to prove it
        p = n // b
        v = hA.view(p * p, b * b)
        for j in range(p):
            for i in range(j):
                v[i + j * p] = float("nan")
    hAux = torch.zeros(tf.tile_qr_t_elems(n, b, ib), dtype=torch.float64).pin_memory() if alg != "chol" else None
    hPiv = torch.zeros(tf.tile_lu_ipiv_elems(n, b), dtype=torch.int32).pin_memory() if alg == "lu" else None
    hInfo = torch.full((1,), 77, dtype=torch.int32)
    tf.tile_factor_host(alg, n, b, ib, hA, hAux, hPiv, hInfo)
    assert int(hInfo.item()) == 0 == gi
    H = hA.numpy()
    if alg == "chol":
        p = n // b
        L1, L2 = oracle.tile_lower_L(H, n, b), oracle.tile_lower_L(G, n, b)
        assert np.array_equal(L1, L2)
    else:
        assert np.array_equal(H, G)
        p = n // b
        for k in range(p):
            for i in range(k if alg == "qr" else k + 1, p):  # T strips i >= k, L strips i > k
                o = (i + k * p) * ib * b
                assert np.array_equal(hAux.numpy()[o:o + ib * b], GA[o:o + ib * b]), (i, k)
        if alg == "lu":
            for k in range(p):
                for i in range(k, p):
                    o = (i + k * p) * b
                    assert np.array_equal(hPiv.numpy()[o:o + b], GP[o:o + b]), (i, k)
