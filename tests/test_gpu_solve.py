"""GPU: solves / applies with the tiled factors and GENP (
PAPER.md:804-891), through the C-ABI, against the oracle.

The solve kernels are compared with the oracle applied to the SAME (GPU-computed) factors,
so the comparison isolates the solve arithmetic (tolerance 1e-10, relative, per the
per-tile bar of north_star); the end-to-end checks are backward errors:
||y - A x||_inf / (||A||_inf ||x||_inf) (the paper's solution backward error)
and ||A - N U||_F / ||A||_F for the explicit N application.  GENP is compared per tile with
the oracle's tiled no-pivot LU on column diagonally dominant inputs (where it is stable)
and bitwise on the exact dyadic pin.
"""
import numpy as np
import pytest

import oracle
import tilegen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from _gpu_util import gpu_factor, gpu_pack, rel, tile_errors  # noqa: E402
from paper_0709_1272_b200 import tilefact as tf  # noqa: E402


def _dev_rhs(Y):
    """numpy (n, nrhs) -> CUDA tensor of shape (nrhs, n) = column-major n x nrhs."""
    return torch.from_numpy(np.ascontiguousarray(Y.T)).cuda()


def _host_rhs(X):
    return X.cpu().numpy().T.copy(order="F")


def _factors(alg, A, b, ib):
    n = A.shape[0]
    T = gpu_pack(A, b)
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    aux = torch.zeros(tf.tile_qr_t_elems(n, b, ib), dtype=torch.float64, device="cuda")
    piv = None
    if alg == "qr":
        tf.tile_qr(n, b, ib, T, aux)
    else:
        piv = torch.zeros(tf.tile_lu_ipiv_elems(n, b), dtype=torch.int32, device="cuda")
        (tf.tile_lu if alg == "lu" else tf.tile_lu_nopiv)(n, b, ib, T, aux, piv, info)
    torch.cuda.synchronize()
    return T, aux, piv, int(info.item())


SIZES = [(512, 128, 32, 3), (768, 256, 32, 1), (1024, 512, 64, 2), (96, 32, 8, 130), (63, 21, 7, 5),
         (256, 256, 32, 1)]


@pytest.mark.parametrize("n,b,ib,nrhs", SIZES)
def test_getrs(n, b, ib, nrhs):
    A = tilegen.normal(n, 21)
    Y = np.asfortranarray(tilegen.normal(n, 22)[:, :nrhs] if nrhs <= n else np.random.default_rng(3).standard_normal((n, nrhs)))
    T, Ls, piv, info = _factors("lu", A, b, ib)
    assert info == 0
    X = _dev_rhs(Y)
    tf.tile_getrs(n, b, ib, T, Ls, piv, X)
    x = _host_rhs(X)
    want = oracle.lu_solve(T.cpu().numpy(), Ls.cpu().numpy(), piv.cpu().numpy(), Y, n, b, ib)
    assert rel(x, want) <= 1e-10, rel(x, want)
    be = np.max(np.abs(Y - A @ x)) / (np.max(np.abs(A).sum(axis=1)) * np.max(np.abs(x)))
    assert be <= 1e-12, be


@pytest.mark.parametrize("n,b,ib,nrhs", SIZES)
def test_ormqr_and_qrs(n, b, ib, nrhs):
    A = tilegen.uniform(n, 23)
    Y = np.asfortranarray(np.random.default_rng(4).standard_normal((n, nrhs)))
    T, Tq, _, _ = _factors("qr", A, b, ib)
    F, G = T.cpu().numpy(), Tq.cpu().numpy()
    X = _dev_rhs(Y)
    tf.tile_ormqr(n, b, ib, T, Tq, X)
    assert rel(_host_rhs(X), oracle.qr_apply(F, G, Y, n, b, ib, trans=True)) <= 1e-12
    X = _dev_rhs(Y)
    tf.tile_qrs(n, b, ib, T, Tq, X)
    x = _host_rhs(X)
    assert rel(x, oracle.qr_solve(F, G, Y, n, b, ib)) <= 1e-10
    be = np.max(np.abs(Y - A @ x)) / (np.max(np.abs(A).sum(axis=1)) * np.max(np.abs(x)))
    assert be <= 1e-13, be


@pytest.mark.parametrize("n,b,ib", [(512, 128, 32), (768, 256, 32), (96, 32, 8), (1024, 512, 64)])
def test_lu_apply_N(n, b, ib):
    A = tilegen.normal(n, 24)
    T, Ls, piv, _ = _factors("lu", A, b, ib)
    F, L, P = T.cpu().numpy(), Ls.cpu().numpy(), piv.cpu().numpy()
    U = oracle.lu_U(F, n, b)
    X = _dev_rhs(U)
    tf.tile_lu_apply_N(n, b, ib, T, Ls, piv, X)
    NU = _host_rhs(X)
    assert rel(NU, oracle.lu_apply_N(F, L, P, U, n, b, ib)) <= 1e-12
    assert np.linalg.norm(A - NU) / np.linalg.norm(A) <= 1e-12


@pytest.mark.parametrize("n,b,ib", [(512, 128, 32), (768, 256, 32), (96, 32, 8), (1024, 512, 64)])
def test_lu_nopiv(n, b, ib):
    A = tilegen.normal(n, 25)
    A[np.diag_indices(n)] = np.abs(A).sum(axis=0) + 1.0  # column diagonally dominant
    T, Ls, piv, info = _factors("nopiv", A, b, ib)
    assert info == 0
    F = oracle.pack(A, b)
    OL, OP, oi = oracle.lu_nopiv(F, n, b, ib)
    G = T.cpu().numpy()
    assert np.array_equal(piv.cpu().numpy(), OP)
    assert max(tile_errors("lu", G, F, n, b).values()) <= 1e-10
    A0, _, _ = tilegen.lu_exact(n, 7)
    T, Ls, piv, _ = _factors("nopiv", A0, b, ib)
    F = oracle.pack(A0, b)
    OL, OP, _ = oracle.lu_nopiv(F, n, b, ib)
    assert np.array_equal(T.cpu().numpy(), F) and np.array_equal(Ls.cpu().numpy(), OL)
