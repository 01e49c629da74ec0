"""GPU: the multi-GPU path run on one B200 through tile_dist_emulate.

tile_dist_emulate runs P*Q ranks in ONE persistent launch (CTA groups), with each rank's
local buffers, receive cache and scheduler state in their own device allocations; the
SEND items' stores into peers' caches and the remote queue pushes use exactly the device
code of the one-process-per-GPU path (tile_dist_factor), only the peer pointers differ
(same-device instead of IPC-mapped).  Results must be bitwise identical to the 1-GPU
factorization (same kernels, per-tile updates chained in k) and within the parity
tolerance of the oracle.
"""
import numpy as np
import pytest

import tilegen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from _gpu_util import gpu_pack, lu_certified, lu_tile_tolerances, oracle_factor, tile_errors  # noqa: E402
from paper_0709_1272_b200 import tilefact as tf  # noqa: E402


def _gen(alg, n, seed):
    return {"chol": tilegen.spd, "qr": tilegen.uniform, "lu": tilegen.normal}[alg](n, seed)


def one_gpu(alg, T, n, b, ib):
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    aux = piv = None
    if alg == "chol":
        tf.tile_chol(n, b, ib, T, info)
    elif alg == "qr":
        aux = torch.zeros(tf.tile_qr_t_elems(n, b, ib), dtype=torch.float64, device="cuda")
        tf.tile_qr(n, b, ib, T, aux)
    else:
        aux = torch.zeros(tf.tile_lu_l_elems(n, b, ib), dtype=torch.float64, device="cuda")
        piv = torch.zeros(tf.tile_lu_ipiv_elems(n, b), dtype=torch.int32, device="cuda")
        tf.tile_lu(n, b, ib, T, aux, piv, info)
    torch.cuda.synchronize()
    return T, aux, piv, int(info.item())


def scatter(alg, T, n, b, ib, P, Q):
    """Global BDL tiles -> per-rank local buffers (include/tilefact.h local layout)."""
    p, R = n // b, P * Q
    ne = tf.tile_dist_local_elems(alg, n, b, ib, P, Q, 0)
    A = [torch.full((ne,), float("nan"), dtype=torch.float64, device="cuda") for _ in range(R)]
    aux = piv = None
    if alg != "chol":
        na = tf.tile_dist_local_elems(alg, n, b, ib, P, Q, 1)
        aux = [torch.zeros(na, dtype=torch.float64, device="cuda") for _ in range(R)]
    if alg == "lu":
        npv = tf.tile_dist_local_elems(alg, n, b, ib, P, Q, 2)
        piv = [torch.zeros(npv, dtype=torch.int32, device="cuda") for _ in range(R)]
    Tv = T.view(p * p, b * b)
    for j in range(p):
        for i in range(p):
            r = tf.tile_dist_owner(i, j, P, Q)
            li = tf.tile_dist_local_index(i, j, p, P, Q)
            A[r].view(-1, b * b)[li].copy_(Tv[i + j * p])
    return A, aux, piv


def gather(alg, A, aux, piv, n, b, ib, P, Q):
    p = n // b
    G = torch.zeros(n * n, dtype=torch.float64, device="cuda")
    GA = torch.zeros(p * p * ib * b, dtype=torch.float64, device="cuda") if aux is not None else None
    GP = torch.zeros(p * p * b, dtype=torch.int32, device="cuda") if piv is not None else None
    for j in range(p):
        for i in range(p):
            r = tf.tile_dist_owner(i, j, P, Q)
            li = tf.tile_dist_local_index(i, j, p, P, Q)
            g = i + j * p
            G.view(-1, b * b)[g].copy_(A[r].view(-1, b * b)[li])
            if GA is not None:
                GA.view(-1, ib * b)[g].copy_(aux[r].view(-1, ib * b)[li])
            if GP is not None:
                GP.view(-1, b)[g].copy_(piv[r].view(-1, b)[li])
    return G, GA, GP


def run_dist(alg, A0, n, b, ib, P, Q):
    A, aux, piv = scatter(alg, A0, n, b, ib, P, Q)
    info = torch.full((1,), 12345, dtype=torch.int32, device="cuda")
    tf.tile_dist_emulate(alg, n, b, ib, P, Q, A, aux, piv, info)
    torch.cuda.synchronize()
    G, GA, GP = gather(alg, A, aux, piv, n, b, ib, P, Q)
    return G, GA, GP, int(info.item())


def lower_mask(n, b):
    """Cholesky: only lower tiles / lower triangles of diagonal tiles are results."""
    p = n // b
    m = torch.zeros(p, p, b, b, dtype=torch.bool)
    tri = torch.tril(torch.ones(b, b, dtype=torch.bool)).t()  # tile stored column-major
    for j in range(p):
        for i in range(p):
            if i > j:
                m[j, i] = True
            elif i == j:
                m[j, i] = tri
    return m.reshape(-1).cuda()


CASES = [
    ("chol", 1024, 128, 32, 1, 1),
    ("chol", 1024, 128, 32, 1, 2),
    ("chol", 1024, 128, 32, 2, 1),
    ("chol", 1024, 128, 32, 2, 2),
    ("chol", 2048, 128, 32, 2, 4),
    ("chol", 1536, 192, 32, 2, 2),   # ragged 128-row items, p not a multiple of Q
    ("qr", 1024, 128, 32, 1, 2),
    ("qr", 1024, 128, 32, 1, 4),
    ("qr", 1280, 128, 32, 1, 8),
    ("qr", 4096, 256, 32, 1, 4),     # config 2 sizes
    ("lu", 1024, 128, 32, 1, 2),
    ("lu", 1152, 128, 32, 1, 4),
    ("lu", 4096, 256, 32, 1, 2),     # config 3 sizes
    ("lu", 2048, 512, 64, 1, 2),     # NEXT-1 tile shape (b = 512, ib = 64), p = 4
    ("qr", 2048, 512, 64, 1, 2),     # config-5 tile shape
]


@pytest.mark.parametrize("alg,n,b,ib,P,Q", CASES)
def test_dist_emulate_bitwise_equals_one_gpu(alg, n, b, ib, P, Q):
    A = _gen(alg, n, 11)
    T0 = gpu_pack(A, b)
    R1, aux1, piv1, info1 = one_gpu(alg, T0.clone(), n, b, ib)
    G, GA, GP, info = run_dist(alg, T0, n, b, ib, P, Q)
    assert info == info1 == 0
    if alg == "chol":
        m = lower_mask(n, b)
        assert torch.equal(G[m], R1[m])
    else:
        assert torch.equal(G, R1)
        p = n // b
        # T / L strips: only (i >= k) strips are written
        sm = torch.zeros(p, p, dtype=torch.bool)
        for k in range(p):
            for i in range(k, p):
                sm[k, i] = True
        sm = sm.reshape(-1).repeat_interleave(ib * b).cuda()
        assert torch.equal(GA[sm], aux1[sm])
        if alg == "lu":
            pm = torch.zeros(p, p, dtype=torch.bool)
            for k in range(p):
                for i in range(k, p):
                    pm[k, i] = True
            pm = pm.reshape(-1).repeat_interleave(b).cuda()
            assert torch.equal(GP[pm], piv1[pm])


@pytest.mark.parametrize("alg,P,Q", [("chol", 2, 2), ("qr", 1, 4), ("lu", 1, 4)])
def test_dist_emulate_matches_oracle(alg, P, Q):
    n, b, ib = 768, 96, 32
    A = _gen(alg, n, 5)
    G, GA, GP, info = run_dist(alg, gpu_pack(A, b), n, b, ib, P, Q)
    O, OA, OP, oi = oracle_factor(alg, A, b, ib)
    assert info == oi == 0
    errs = tile_errors(alg, G.cpu().numpy(), O, n, b)
    if alg != "lu":
        assert max(errs.values()) <= 1e-10
    else:
        # the C5 reading: max(1e-10, 10 sigma_t), the perturbed oracle keeping the pivots
        c = lu_certified(n, b, ib, 5)
        assert c["seed"] == 5 and np.array_equal(c["O"], O)
        tol, sig = lu_tile_tolerances(c, n, b)
        for key, e in errs.items():
            assert e <= tol[key], (key, e, sig[key])
    if alg == "lu":
        p = n // b
        Gp = GP.cpu().numpy()
        for k in range(p):
            for i in range(k, p):
                o = (i + k * p) * b
                assert np.array_equal(Gp[o:o + b], OP[o:o + b])


def test_dist_emulate_repeated_calls_and_fewer_ctas():
    """Epoch-tagged barriers: back-to-back calls on the same handles, and a small grid."""
    alg, n, b, ib, P, Q = "qr", 1024, 128, 32, 1, 4
    A = _gen(alg, n, 2)
    T0 = gpu_pack(A, b)
    ref = run_dist(alg, T0, n, b, ib, P, Q)
    for ctas in (0, 8, 13):
        tf.tile_set_ctas(ctas)
        try:
            for _ in range(2):
                G, GA, _, info = run_dist(alg, T0, n, b, ib, P, Q)
                assert info == 0 and torch.equal(G, ref[0]) and torch.equal(GA, ref[1])
        finally:
            tf.tile_set_ctas(0)


def test_dist_emulate_chol_not_spd_reports_info_and_stops():
    n, b, ib, P, Q = 1024, 128, 32, 2, 2
    A = tilegen.spd(n, 1)
    A[700, 700] = -5.0  # leading minor of order 701 is not positive definite
    T0 = gpu_pack(A, b)
    _, _, _, info1 = one_gpu("chol", T0.clone(), n, b, ib)
    _, _, _, info = run_dist("chol", T0, n, b, ib, P, Q)
    assert info1 == 701 and info == info1
    # the handles are reusable after an aborted run
    A2 = tilegen.spd(n, 2)
    T2 = gpu_pack(A2, b)
    R1, _, _, _ = one_gpu("chol", T2.clone(), n, b, ib)
    G, _, _, info = run_dist("chol", T2, n, b, ib, P, Q)
    m = lower_mask(n, b)
    assert info == 0 and torch.equal(G[m], R1[m])


@pytest.mark.parametrize("alg", ["chol", "qr", "lu"])
def test_dist_handle_single_rank_equals_one_gpu(alg):
    """tile_dist_open/factor/close (the one-process-per-GPU API) with a 1 x 1 grid."""
    n, b, ib = 1024, 128, 32
    A = _gen(alg, n, 4)
    T0 = gpu_pack(A, b)
    R1, aux1, piv1, _ = one_gpu(alg, T0.clone(), n, b, ib)
    h = tf.DistHandle(alg, n, b, ib, 1, 1, 0)
    Aloc, aux, piv = scatter(alg, T0, n, b, ib, 1, 1)
    info = torch.full((1,), 7, dtype=torch.int32, device="cuda")
    for _ in range(2):  # repeated calls: epoch-tagged barriers
        Aloc, aux, piv = scatter(alg, T0, n, b, ib, 1, 1)
        h.factor(Aloc[0], None if aux is None else aux[0], None if piv is None else piv[0], info)
        torch.cuda.synchronize()
        assert int(info.item()) == 0
        if alg == "chol":
            m = lower_mask(n, b)
            assert torch.equal(Aloc[0][m], R1[m])
        else:
            assert torch.equal(Aloc[0], R1)
    h.close()


def test_bench_dist_runner_single_rank():
    """bench.py's multi-GPU runner end to end with a 1-rank process group (gloo)."""
    import os
    import sys
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        for c in (1, 2, 3):
            cfg = dict(bench.CONFIGS[c])
            res = bench.run_dist_device(tf, torch, cfg, 2, 1, 0, 1)
            assert res["info"] == 0 and len(res["ms"]) == 2 and res["grid"] == "1x1"
            assert res["e2e"]["h2d"] == cfg["n"] ** 2 * 8
    finally:
        dist.destroy_process_group()
