"""GPU parity of the rectangular tiled QR / LU (Algorithms 2 / 3 on a
p x q tiled matrix) against the oracle's o_qr_mn / o_lu_mn.

Tall, wide, tall-skinny and p x q with a ragged slab path (b = 96) are covered.  Same bar
as the square parity tests: per tile <= 1e-10 relative Frobenius for QR (T strips too),
LU pivots bit-identical with the per-tile C5 reading (the perturbed oracle run must keep
the pivots), and the reconstructions (Q R = A, N U = A) at the square-case bounds.
"""
import numpy as np
import pytest

import oracle
import tilegen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from _gpu_util import rel, to_dev_colmajor  # noqa: E402
from paper_0709_1272_b200 import tilefact as tf  # noqa: E402

SHAPES = [(768, 512, 256, 32), (512, 768, 256, 32), (1024, 256, 128, 32), (256, 1024, 128, 32),
          (1536, 1024, 512, 64), (96 * 3, 96 * 2, 96, 32), (63, 42, 21, 7)]


def _mat(m, n, seed, gen):
    return np.asfortranarray(gen(max(m, n), seed)[:m, :n])


def _pack(A, b):
    m, n = A.shape
    D = to_dev_colmajor(A)
    T = torch.empty(m * n, dtype=torch.float64, device="cuda")
    tf.tile_pack(m, n, b, D, T)
    return T


def _tiles(F, m, n, b):
    p, q = m // b, n // b
    return {(i, j): F[(i + j * p) * b * b:(i + j * p + 1) * b * b] for j in range(q) for i in range(p)}


@pytest.mark.parametrize("m,n,b,ib", SHAPES)
def test_qr_mn_parity(m, n, b, ib):
    A = _mat(m, n, 31, tilegen.uniform)
    T = _pack(A, b)
    Tq = torch.zeros(tf.tile_mn_aux_elems(m, n, b, ib), dtype=torch.float64, device="cuda")
    tf.tile_qr_mn(m, n, b, ib, T, Tq)
    torch.cuda.synchronize()
    G, GT = T.cpu().numpy(), Tq.cpu().numpy()
    F = oracle.pack(A, b)
    OT = oracle.qr_mn(F, m, n, b, ib)
    tg, to = _tiles(G, m, n, b), _tiles(F, m, n, b)
    worst = max(rel(tg[k], to[k]) for k in to)
    assert worst <= 1e-10, worst
    assert rel(GT, OT) <= 1e-10
    k = min(m, n)
    R = oracle.upper_mn(G, m, n, b)
    Rk = np.vstack([R[:k], np.zeros((m - k, n))]) if m > k else R[:k]
    QR = oracle.qr_apply_mn(G, GT, Rk, m, n, b, ib)
    assert np.linalg.norm(QR - A) / np.linalg.norm(A) <= 1e-13


@pytest.mark.parametrize("m,n,b,ib", SHAPES)
def test_lu_mn_parity(m, n, b, ib):
    A = _mat(m, n, 32, tilegen.normal)
    T = _pack(A, b)
    Ls = torch.zeros(tf.tile_mn_aux_elems(m, n, b, ib), dtype=torch.float64, device="cuda")
    piv = torch.zeros(tf.tile_mn_ipiv_elems(m, n, b), dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    tf.tile_lu_mn(m, n, b, ib, T, Ls, piv, info)
    torch.cuda.synchronize()
    G, GL, Gp = T.cpu().numpy(), Ls.cpu().numpy(), piv.cpu().numpy()
    F = oracle.pack(A, b)
    OL, Op, oi = oracle.lu_mn(F, m, n, b, ib)
    assert int(info.item()) == oi == 0
    # C5: the oracle's own spread under a 2^-52 perturbation, same pivots required
    r = np.random.default_rng(7)
    Fp = oracle.pack(A * (1.0 + 2.0 ** -52 * r.standard_normal(A.shape)), b)
    _, Pp, _ = oracle.lu_mn(Fp, m, n, b, ib)
    assert np.array_equal(Pp, Op), "seed is pivot-fragile"
    assert np.array_equal(Gp, Op)
    tg, to, tp = _tiles(G, m, n, b), _tiles(F, m, n, b), _tiles(Fp, m, n, b)
    for key in to:
        assert rel(tg[key], to[key]) <= max(1e-10, 10 * rel(tp[key], to[key])), key
    U = oracle.upper_mn(G, m, n, b)
    NU = oracle.lu_apply_N_mn(G, GL, Gp, U, m, n, b, ib)
    ro = np.linalg.norm(A - oracle.lu_apply_N_mn(F, OL, Op, oracle.upper_mn(F, m, n, b), m, n, b, ib))
    assert np.linalg.norm(A - NU) <= max(1e-12 * np.linalg.norm(A), 2 * ro)
