"""Seeded synthetic input generators — shared by the oracle tests and the CUDA path.

Holds none of the method's arithmetic: only the input recipes of BASELINE.json's configs
(SURVEY.md §8(d) "Concrete synthetic inputs", §8(c) C0) and the exact-pin matrices of
SURVEY.md §8(c) C5.  Every generator is a pure function of (n, seed) built on numpy's
counter-based Philox bit generator, so the same seed gives the same bytes everywhere.
Outputs are dense column-major (Fortran-order) float64 arrays; conversion to the tile
layout is done separately by each side (oracle.pack / the library's tile_pack).

For the n=32768 configs, ``*_torch`` variants build the same distributions directly in
device memory with torch's CUDA generator (8 GiB per matrix is too slow to stage from
numpy); those large inputs are only ever checked through properties (residual probes),
never element by element against the oracle.
"""
from __future__ import annotations

import numpy as np


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=int(seed) & (2**64 - 1)))


def uniform(n: int, seed: int, lo: float = -0.5, hi: float = 0.5, m: int | None = None) -> np.ndarray:
    """i.i.d. U[lo, hi) (configs 2 and 5 use [-0.5, 0.5)). u in [0,1) with 53-bit
    resolution; lo + (hi-lo)*u is exact for the two ranges used here."""
    m = n if m is None else m
    u = _rng(seed).random((m, n))
    return np.asfortranarray(lo + (hi - lo) * u)


def normal(n: int, seed: int, m: int | None = None) -> np.ndarray:
    """i.i.d. N(0,1) (config 3; the paper's randn)."""
    m = n if m is None else m
    return np.asfortranarray(_rng(seed).standard_normal((m, n)))


def spd(n: int, seed: int) -> np.ndarray:
    """A = M M^T / n + n I with M i.i.d. U[-1,1] (configs 1 and 4).  The product is
    rounded once here and the same bytes go to both sides (C0)."""
    M = uniform(n, seed, -1.0, 1.0)
    A = (M @ M.T) / n
    A[np.diag_indices(n)] += n
    return np.asfortranarray(A)


# ------------------------------------------------------------------ exact pins (C5)

def chol_exact(n: int, seed: int):
    """A = L0 L0^T with L0 integer in [-4,4] strictly below the diagonal and diagonal in
    {1,2,4}.  All intermediate values of any Cholesky ordering are integers < 2^53, so
    L = L0 exactly."""
    r = _rng(seed)
    L0 = np.tril(r.integers(-4, 5, size=(n, n)), -1).astype(np.int64)
    L0[np.diag_indices(n)] = r.choice([1, 2, 4], size=n)
    A = L0 @ L0.T
    assert np.abs(A).max() < 2**52
    return np.asfortranarray(A.astype(np.float64)), np.asfortranarray(L0.astype(np.float64))


def lu_exact(n: int, seed: int):
    """A = L0 U0, L0 unit lower with multiples of 1/4 of magnitude <= 3/4, U0 integer in
    [-3,3] above the diagonal and diagonal in {+-2, +-4}.  No pivot ever swaps (every
    candidate below the pivot is < |pivot|) and all values are dyadic with few bits, so
    any elimination order reproduces U = U0 and the multipliers = L0 exactly."""
    r = _rng(seed)
    L4 = np.tril(r.integers(-3, 4, size=(n, n)), -1).astype(np.int64)  # 4*L0 strictly lower
    L4[np.diag_indices(n)] = 4
    U0 = np.triu(r.integers(-3, 4, size=(n, n)), 1).astype(np.int64)
    U0[np.diag_indices(n)] = r.choice([-4, -2, 2, 4], size=n)
    A4 = L4 @ U0  # = 4 * A, exact in int64
    assert np.abs(A4).max() < 2**50
    A = A4.astype(np.float64) / 4.0
    return (np.asfortranarray(A), np.asfortranarray(L4.astype(np.float64) / 4.0),
            np.asfortranarray(U0.astype(np.float64)))


def qr_perm(n: int, seed: int):
    """Scaled permutation P D with entries +-{1,2,4}: every Householder step is exact
    (tau in {0,1}), |R| = |D| on the diagonal and 0 elsewhere (C5)."""
    r = _rng(seed)
    perm = r.permutation(n)
    d = r.choice([1.0, 2.0, 4.0], size=n) * r.choice([-1.0, 1.0], size=n)
    A = np.zeros((n, n))
    A[perm, np.arange(n)] = d
    return np.asfortranarray(A), d


def qr_upper(n: int, seed: int):
    """Upper-triangular input: every reflector is trivial (tau = 0) and R = A bitwise."""
    r = _rng(seed)
    A = np.triu(r.integers(-8, 9, size=(n, n)).astype(np.float64))
    A[np.diag_indices(n)] = r.choice([1.0, 3.0, -2.0, 5.0], size=n)
    return np.asfortranarray(A)


def hadamard(n: int) -> np.ndarray:
    """Sylvester-Hadamard matrix (n a power of two): H^T H = n I, so |R| = sqrt(n) I."""
    H = np.ones((1, 1))
    while H.shape[0] < n:
        H = np.block([[H, H], [H, -H]])
    assert H.shape[0] == n
    return np.asfortranarray(H)


# ------------------------------------------------------------------ large configs on device

def uniform_torch(n: int, seed: int, lo: float, hi: float, device):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    u = torch.rand((n, n), dtype=torch.float64, generator=g, device=device)
    return u.mul_(hi - lo).add_(lo)


def normal_torch(n: int, seed: int, device):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return torch.randn((n, n), dtype=torch.float64, generator=g, device=device)


def spd_torch(n: int, seed: int, device):
    """Same recipe as ``spd`` for the n=32768 configs, built on the device.  Returned as
    a torch tensor whose *column-major* reading is the matrix (it is symmetric anyway)."""
    import torch
    M = uniform_torch(n, seed, -1.0, 1.0, device)
    A = torch.matmul(M, M.T)
    del M
    A.div_(n)
    A.diagonal().add_(n)
    return A
