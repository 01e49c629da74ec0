"""GPU: the slab-level task graph (tile_set_slab_dag) gives results bitwise
identical to the paper's tile-level graph: every tile sees the same
kernel operations in the same order, only the granularity of the dependencies changes.
Factors, T / L strips, pivots and info are compared bit for bit, over square and
rectangular tile grids, ib = 32 and 64, and a singular LU (info from a slab task)."""
import numpy as np
import pytest
import torch

import tilegen
from _gpu_util import gpu_factor, gpu_pack
from paper_0709_1272_b200 import tilefact as tf

pytestmark = pytest.mark.gpu


def _both(fn):
    out = []
    for on in (0, 1):
        tf.tile_set_slab_dag(on)
        try:
            out.append(fn())
        finally:
            tf.tile_set_slab_dag(-1)
    return out


@pytest.mark.parametrize("alg,n,b,ib,seed", [("qr", 1024, 256, 32, 0), ("lu", 1024, 256, 32, 1),
                                             ("qr", 1536, 512, 64, 2), ("lu", 1536, 512, 64, 3),
                                             ("qr", 640, 128, 32, 4), ("lu", 640, 128, 64, 5),
                                             ("lu", 2048, 256, 64, 6),
                                             # panel-level Cholesky graph (b a multiple of 128, >= 256)
                                             ("chol", 2048, 512, 64, 7), ("chol", 1280, 256, 32, 8),
                                             ("chol", 1152, 384, 32, 9), ("chol", 2048, 1024, 64, 10),
                                             ("chol", 1920, 640, 32, 13), ("chol", 2304, 1152, 32, 14)])
def test_slab_dag_bitwise_equals_tile_dag(alg, n, b, ib, seed):
    A = {"chol": tilegen.spd, "qr": tilegen.uniform, "lu": tilegen.normal}[alg](n, seed)
    (G0, X0, P0, i0), (G1, X1, P1, i1) = _both(lambda: gpu_factor(alg, A, b, ib))
    assert np.array_equal(G0.view(np.int64), G1.view(np.int64))
    if alg != "chol":
        assert np.array_equal(X0.view(np.int64), X1.view(np.int64))
    if alg == "lu":
        assert np.array_equal(P0, P1)
    assert i0 == i1 == 0


@pytest.mark.parametrize("n,b,tile_min", [(4096, 512, 1), (3072, 256, 10), (3072, 384, 3)])
def test_panel_dag_whole_tile_gemm_bitwise(n, b, tile_min):
    """Whole-tile GEMM items (one slice stream over the nr x nr sub-tile products) give the
    same bits as the strip items and as the tile-level graph."""
    A = tilegen.spd(n, 12)
    outs = []
    for fine, tm in ((0, -1), (1, 0), (1, tile_min)):
        tf.tile_set_slab_dag(fine)
        tf.tile_set_gemm_tile_min(tm)
        try:
            outs.append(gpu_factor("chol", A, b, 32))
        finally:
            tf.tile_set_slab_dag(-1)
            tf.tile_set_gemm_tile_min(-1)
    for G, _, _, info in outs[1:]:
        assert info == 0
        assert np.array_equal(G.view(np.int64), outs[0][0].view(np.int64))


def test_panel_dag_schedule_independent():
    """The panel-level Cholesky graph gives the same bits for any grid size, priority policy
    and run (several CTAs now work inside one POTRF / TRSM; every block still sees its
    operations in one fixed order), and a one-CTA grid completes (no CTA ever waits for a
    specific task)."""
    n, b = 2048, 512
    A = tilegen.spd(n, 15)
    ref = gpu_factor("chol", A, b, 64)[0].view(np.int64)
    try:
        for ctas, policy in ((1, 1), (3, 0), (7, 1), (40, 0), (148, 0), (0, 1)):
            tf.tile_set_ctas(ctas)
            tf.tile_set_policy(policy)
            for _ in range(2):
                G, _, _, info = gpu_factor("chol", A, b, 64)
                assert info == 0 and np.array_equal(G.view(np.int64), ref), (ctas, policy)
    finally:
        tf.tile_set_ctas(0)
        tf.tile_set_policy(1)


@pytest.mark.parametrize("col", [70, 300, 512 + 130, 1023])
def test_panel_dag_chol_not_spd_info(col):
    """A non-positive pivot inside a later 128-column panel / tile: info comes from the
    panel-level diagonal-block task and equals the tile-level graph's and the oracle's."""
    import oracle
    n, b = 1024, 512
    A = tilegen.spd(n, 11)
    A[col, col] = -1e6
    (_, _, _, i0), (_, _, _, i1) = _both(lambda: gpu_factor("chol", A, b, 64))
    F = oracle.pack(A, b)
    assert i0 == i1 == oracle.chol(F, n, b) == col + 1


def test_slab_dag_singular_lu_info():
    n, b, ib = 768, 256, 32
    A = tilegen.normal(n, 7)
    A[:, 300] = 0.0  # a zero column inside slab 1 of tile column 1
    (G0, _, P0, i0), (G1, _, P1, i1) = _both(lambda: gpu_factor("lu", A, b, ib))
    assert i0 == i1 and i0 > 0
    assert np.array_equal(P0, P1)


@pytest.mark.parametrize("alg,m,n,b,ib", [("qr", 1536, 768, 256, 32), ("lu", 1536, 768, 256, 32),
                                          ("qr", 768, 1536, 256, 64), ("lu", 1024, 512, 128, 32)])
def test_slab_dag_rectangular_bitwise(alg, m, n, b, ib):
    rng = np.random.default_rng(11)
    A = rng.uniform(-0.5, 0.5, (m, n)) if alg == "qr" else rng.standard_normal((m, n))

    def run():
        T = gpu_pack(A, b)
        aux = torch.zeros(tf.tile_mn_aux_elems(m, n, b, ib), dtype=torch.float64, device="cuda")
        if alg == "qr":
            tf.tile_qr_mn(m, n, b, ib, T, aux)
            piv = None
        else:
            piv = torch.zeros(tf.tile_mn_ipiv_elems(m, n, b), dtype=torch.int32, device="cuda")
            info = torch.zeros(1, dtype=torch.int32, device="cuda")
            tf.tile_lu_mn(m, n, b, ib, T, aux, piv, info)
        torch.cuda.synchronize()
        return T.cpu().numpy(), aux.cpu().numpy(), None if piv is None else piv.cpu().numpy()

    (G0, X0, P0), (G1, X1, P1) = _both(run)
    assert np.array_equal(G0.view(np.int64), G1.view(np.int64))
    assert np.array_equal(X0.view(np.int64), X1.view(np.int64))
    if P0 is not None:
        assert np.array_equal(P0, P1)
