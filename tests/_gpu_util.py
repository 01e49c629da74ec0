"""Helpers for the GPU parity tests: run the CUDA path through the C-ABI binding and the
oracle on the same seeded inputs, and compare tile by tile.

Tolerances (BASELINE north_star): per tile ||G - O||_F / ||O||_F <= 1e-10
for Cholesky and QR; LU pivots bit-exact and per-tile relative error <= max(1e-10,
10 * sigma_t) where sigma_t is the oracle's own self-spread under a 2^-52 relative input
perturbation (SURVEY §8(c) C5 reading).
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_0709_1272_b200 import tilefact as tf


def to_dev_colmajor(A: np.ndarray) -> torch.Tensor:
    """Column-major device copy of a dense matrix (1-D tensor)."""
    return torch.from_numpy(np.asfortranarray(A).ravel(order="F").copy()).cuda()


def gpu_pack(A: np.ndarray, b: int) -> torch.Tensor:
    m, n = A.shape
    D = to_dev_colmajor(A)
    T = torch.empty(m * n, dtype=torch.float64, device="cuda")
    tf.tile_pack(m, n, b, D, T)
    return T


def gpu_factor(alg: str, A: np.ndarray, b: int, ib: int):
    """Returns (tiles np, aux np or None, ipiv np or None, info int)."""
    n = A.shape[0]
    T = gpu_pack(A, b)
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
    return (T.cpu().numpy(), None if aux is None else aux.cpu().numpy(),
            None if piv is None else piv.cpu().numpy(), int(info.item()))


def oracle_factor(alg: str, A: np.ndarray, b: int, ib: int):
    n = A.shape[0]
    F = oracle.pack(A, b)
    if alg == "chol":
        info = oracle.chol(F, n, b)
        return F, None, None, info
    if alg == "qr":
        T = oracle.qr(F, n, b, ib)
        return F, T, None, 0
    Ls, piv, info = oracle.lu(F, n, b, ib)
    return F, Ls, piv, info


def tile(F, p, b, i, j):
    o = (i + j * p) * b * b
    return F[o:o + b * b].reshape(b, b).T  # (r, c)


def strip(S, p, b, ib, i, k):
    o = (i + k * p) * ib * b
    return S[o:o + ib * b].reshape(b, ib).T  # (r in ib, c in b)


def rel(G, O):
    no = np.linalg.norm(O)
    d = np.linalg.norm(G - O)
    return d / no if no > 0 else d


def tile_errors(alg, G, O, n, b):
    """Per-tile relative Frobenius errors over the tiles that hold results."""
    p = n // b
    errs = {}
    for j in range(p):
        for i in range(p):
            if alg == "chol" and i < j:
                continue
            g, o = tile(G, p, b, i, j), tile(O, p, b, i, j)
            if alg == "chol" and i == j:
                g, o = np.tril(g), np.tril(o)
            errs[(i, j)] = rel(g, o)
    return errs


# ------------------------------------------------------------------ LU reference with C5 certification

MARGIN_MIN = 100.0   # parity runs use seeds whose pivot margin is >= 100


def lu_certified(n, b, ib, seed, gen=None, tries=6):
    """Oracle LU of a seeded N(0,1) matrix plus the C5 self-spread run.

    The oracle is re-run on A o (1 + 2^-52 xi), xi ~ N(0,1).  The
    reading requires that perturbed run to keep the SAME pivots; if it does not, or the
    pivot margin (oracle.pivot_margin) is below MARGIN_MIN, the seed is pivot-fragile:
    it is reported and the next seed (seed + 1000) is used.  Returns a dict with the
    accepted seed, the input, the oracle factors, the perturbed factors, the margin and
    the list of rejected (seed, reason) pairs."""
    import tilegen
    gen = gen or tilegen.normal
    rejected = []
    for t in range(tries):
        sd = seed + 1000 * t
        A = gen(n, sd)
        F = oracle.pack(A, b)
        OL, Op, oi, dec = oracle.lu_decisions(F, n, b, ib)
        r = np.random.default_rng(1234 + sd)
        Ap = A * (1.0 + 2.0 ** -52 * r.standard_normal(A.shape))
        Fp = oracle.pack(Ap, b)
        PL, Pp, _, decp = oracle.lu_decisions(Fp, n, b, ib)
        if not np.array_equal(Pp, Op):
            rejected.append((sd, "perturbed oracle flips a pivot"))
            continue
        m = oracle.pivot_margin(dec, decp)
        if m < MARGIN_MIN:
            rejected.append((sd, f"pivot margin {m:.3g} < {MARGIN_MIN}"))
            continue
        print(f"[C5] n={n} b={b} ib={ib}: seed {sd} pivot margin {m:.3g}; rejected {rejected}")
        return dict(seed=sd, A=A, O=F, OL=OL, Op=Op, info=oi, P=Fp, PL=PL, margin=m, rejected=rejected)
    raise AssertionError(f"no pivot-robust seed found: {rejected}")


def lu_tile_tolerances(cert, n, b):
    """Per-tile tolerance max(1e-10, 10 sigma_t), sigma_t = the oracle's own spread."""
    sig = tile_errors("lu", cert["P"], cert["O"], n, b)
    return {k: max(1e-10, 10 * v) for k, v in sig.items()}, sig
