"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product package
(``paper_0709_1272_b200``) never imports it, and the two share no code.

Thin ctypes wrapper over ``oracle.c`` (plain-loop FP64 kernels written in the order of
the paper's Algorithms 1-3; see the header of
oracle.c for per-function citations).  Arrays are numpy float64 / int32, Fortran
(column-major) order for dense matrices, flat for tile (BDL) storage.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# kind ids for o_kernel_flops (same numbering as the task kinds documented in DESIGN.md)
KINDS = ["potrf", "trsm", "syrk", "gemm", "geqrt", "larfb", "tsqrt", "ssrfb",
         "getrf", "gessm", "tstrf", "ssssm"]


def build(force: bool = False) -> str:
    """Compile oracle.c with -O2 -ffp-contract=off (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-std=c11", "-o", tmp, _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, dp, ip = ctypes.c_int64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32)
        sig = {
            "o_pack": (None, [i64, i64, i64, dp, dp]),
            "o_unpack": (None, [i64, i64, i64, dp, dp]),
            "o_potrf": (ctypes.c_int, [i64, dp]),
            "o_trsm": (None, [i64, dp, dp]),
            "o_syrk": (None, [i64, dp, dp]),
            "o_gemm_nt": (None, [i64, dp, dp, dp]),
            "o_chol": (ctypes.c_int, [i64, i64, dp]),
            "o_geqrt": (None, [i64, i64, dp, dp]),
            "o_larfb": (None, [i64, i64, dp, dp, dp]),
            "o_tsqrt": (None, [i64, i64, dp, dp, dp]),
            "o_ssrfb": (None, [i64, i64, dp, dp, dp, dp]),
            "o_qr": (None, [i64, i64, i64, dp, dp]),
            "o_qr_apply": (None, [i64, i64, i64, dp, dp, dp, i64, ctypes.c_int]),
            "o_getrf": (None, [i64, i64, dp, ip, ctypes.POINTER(ctypes.c_int)]),
            "o_gessm": (None, [i64, i64, dp, ip, dp]),
            "o_tstrf": (None, [i64, i64, dp, dp, dp, ip, ctypes.POINTER(ctypes.c_int)]),
            "o_ssssm": (None, [i64, i64, dp, dp, ip, dp, dp]),
            "o_lu": (ctypes.c_int, [i64, i64, i64, dp, dp, ip]),
            "o_lu_apply_N": (None, [i64, i64, i64, dp, dp, ip, dp, i64]),
            "o_ref_chol": (ctypes.c_int, [i64, dp]),
            "o_ref_qr": (None, [i64, dp, dp]),
            "o_ref_gepp": (ctypes.c_int, [i64, dp, ip]),
            "o_ref_gewp": (ctypes.c_int, [i64, dp, ip]),
            "o_chol_residual": (ctypes.c_double, [i64, dp, dp]),
            "o_kernel_flops": (ctypes.c_double, [ctypes.c_int, ctypes.c_double, ctypes.c_double]),
            "o_decisions_arm": (None, [dp, i64]),
            "o_factor_par": (ctypes.c_int, [ctypes.c_int, i64, i64, i64, dp, dp, ip, ctypes.c_int]),
            "o_qr_mn": (None, [i64, i64, i64, i64, dp, dp]),
            "o_lu_mn": (ctypes.c_int, [i64, i64, i64, i64, dp, dp, ip]),
            "o_qr_apply_mn": (None, [i64, i64, i64, i64, dp, dp, dp, i64, ctypes.c_int]),
            "o_lu_apply_N_mn": (None, [i64, i64, i64, i64, dp, dp, ip, dp, i64]),
            "o_lu_nopiv": (ctypes.c_int, [i64, i64, i64, dp, dp, ip]),
            "o_ref_genp": (ctypes.c_int, [i64, dp]),
            "o_trsm_upper_bdl": (None, [i64, i64, dp, dp, i64, i64]),
            "o_lu_solve": (None, [i64, i64, i64, dp, dp, ip, dp, i64, i64]),
            "o_decisions_count": (i64, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and (a.flags.f_contiguous or a.flags.c_contiguous and a.ndim == 1)
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


# ---------------------------------------------------------------- layout

def pack(dense: np.ndarray, b: int) -> np.ndarray:
    """Dense column-major (m x n) -> flat BDL tile storage."""
    d = np.asfortranarray(dense, dtype=np.float64)
    m, n = d.shape
    out = np.empty(m * n, dtype=np.float64)
    lib().o_pack(m, n, b, _d(d), _d(out))
    return out


def unpack(tiles: np.ndarray, m: int, n: int, b: int) -> np.ndarray:
    out = np.empty((m, n), dtype=np.float64, order="F")
    lib().o_unpack(m, n, b, _d(np.ascontiguousarray(tiles)), _d(out))
    return out


# ---------------------------------------------------------------- tile kernels (in place)

def potrf(A: np.ndarray) -> int:
    return lib().o_potrf(A.shape[0], _d(A))


def trsm(L, A):
    lib().o_trsm(A.shape[0], _d(L), _d(A))


def syrk(A, C):
    lib().o_syrk(C.shape[0], _d(A), _d(C))


def gemm_nt(A, B, C):
    lib().o_gemm_nt(C.shape[0], _d(A), _d(B), _d(C))


def geqrt(A, ib):
    b = A.shape[0]
    T = np.zeros((ib, b), dtype=np.float64, order="F")
    lib().o_geqrt(b, ib, _d(A), _d(T))
    return T


def larfb(V, T, C, ib):
    lib().o_larfb(C.shape[0], ib, _d(V), _d(T), _d(C))


def tsqrt(R, A, ib):
    b = A.shape[0]
    T = np.zeros((ib, b), dtype=np.float64, order="F")
    lib().o_tsqrt(b, ib, _d(R), _d(A), _d(T))
    return T


def ssrfb(V, T, R, A, ib):
    lib().o_ssrfb(A.shape[0], ib, _d(V), _d(T), _d(R), _d(A))


def getrf(A, ib):
    b = A.shape[0]
    piv = np.zeros(b, dtype=np.int32)
    info = ctypes.c_int(0)
    lib().o_getrf(b, ib, _d(A), _i(piv), ctypes.byref(info))
    return piv, info.value


def gessm(L, piv, A, ib):
    lib().o_gessm(A.shape[0], ib, _d(L), _i(piv), _d(A))


def tstrf(U, A, ib):
    b = A.shape[0]
    Ls = np.zeros((ib, b), dtype=np.float64, order="F")
    piv = np.zeros(b, dtype=np.int32)
    info = ctypes.c_int(0)
    lib().o_tstrf(b, ib, _d(U), _d(A), _d(Ls), _i(piv), ctypes.byref(info))
    return Ls, piv, info.value


def ssssm(L, Ls, piv, U, A, ib):
    lib().o_ssssm(A.shape[0], ib, _d(L), _d(Ls), _i(piv), _d(U), _d(A))


# ---------------------------------------------------------------- drivers (BDL in place)

def chol(tiles: np.ndarray, n: int, b: int) -> int:
    return lib().o_chol(n, b, _d(tiles))


def qr(tiles: np.ndarray, n: int, b: int, ib: int) -> np.ndarray:
    p = n // b
    T = np.zeros(p * p * ib * b, dtype=np.float64)
    lib().o_qr(n, b, ib, _d(tiles), _d(T))
    return T


def lu(tiles: np.ndarray, n: int, b: int, ib: int):
    p = n // b
    Ls = np.zeros(p * p * ib * b, dtype=np.float64)
    piv = np.zeros(p * p * b, dtype=np.int32)
    info = lib().o_lu(n, b, ib, _d(tiles), _d(Ls), _i(piv))
    return Ls, piv, info


# ---------------------------------------------------------------- rectangular (NEXT-4)

def qr_mn(tiles: np.ndarray, m: int, n: int, b: int, ib: int) -> np.ndarray:
    """Algorithm 2 on an m x n matrix (p x q tiles).  Returns T strips
    (p * min(p, q) strips of ib x b)."""
    p, q = m // b, n // b
    T = np.zeros(p * min(p, q) * ib * b, dtype=np.float64)
    lib().o_qr_mn(m, n, b, ib, _d(tiles), _d(T))
    return T


def lu_mn(tiles: np.ndarray, m: int, n: int, b: int, ib: int):
    """Algorithm 3 on an m x n matrix (p x q tiles)."""
    p, q = m // b, n // b
    Ls = np.zeros(p * min(p, q) * ib * b, dtype=np.float64)
    piv = np.zeros(p * min(p, q) * b, dtype=np.int32)
    info = lib().o_lu_mn(m, n, b, ib, _d(tiles), _d(Ls), _i(piv))
    return Ls, piv, info


def qr_apply_mn(F, T, X, m, n, b, ib, trans=False):
    X = np.asfortranarray(X, dtype=np.float64).copy(order="F")
    X = X.reshape(-1, 1, order="F") if X.ndim == 1 else X
    lib().o_qr_apply_mn(m, n, b, ib, _d(np.ascontiguousarray(F)), _d(np.ascontiguousarray(T)), _d(X),
                        X.shape[1], 1 if trans else 0)
    return X


def lu_apply_N_mn(F, Ls, piv, X, m, n, b, ib):
    X = np.asfortranarray(X, dtype=np.float64).copy(order="F")
    X = X.reshape(-1, 1, order="F") if X.ndim == 1 else X
    lib().o_lu_apply_N_mn(m, n, b, ib, _d(np.ascontiguousarray(F)), _d(np.ascontiguousarray(Ls)),
                          _i(np.ascontiguousarray(piv)), _d(X), X.shape[1])
    return X


def upper_mn(F, m, n, b):
    """R / U of an m x n factorization: the upper trapezoid of the unpacked matrix."""
    return np.triu(unpack(F, m, n, b))


def lu_nopiv(tiles: np.ndarray, n: int, b: int, ib: int):
    """GENP in tiled form (Algorithm 3 with every pivot kept)."""
    p = n // b
    Ls = np.zeros(p * p * ib * b, dtype=np.float64)
    piv = np.zeros(p * p * b, dtype=np.int32)
    info = lib().o_lu_nopiv(n, b, ib, _d(tiles), _d(Ls), _i(piv))
    return Ls, piv, info


def ref_genp(A):
    """Unblocked GENP (textbook): returns (LU packed, info)."""
    A = np.asfortranarray(A, dtype=np.float64).copy(order="F")
    info = lib().o_ref_genp(A.shape[0], _d(A))
    return A, info


def _rhs(X):
    X = np.asfortranarray(X, dtype=np.float64).copy(order="F")
    return X.reshape(-1, 1, order="F") if X.ndim == 1 else X


def trsm_upper(F, X, n, b):
    """X <- U^{-1} X with U the upper triangle of BDL F (back substitution)."""
    X = _rhs(X)
    lib().o_trsm_upper_bdl(n, b, _d(np.ascontiguousarray(F)), _d(X), X.shape[1], X.shape[0])
    return X


def lu_solve(F, Ls, piv, X, n, b, ib):
    """X <- A^{-1} X = U^{-1} N^{-1} X with the factors of Algorithm 3."""
    X = _rhs(X)
    lib().o_lu_solve(n, b, ib, _d(np.ascontiguousarray(F)), _d(np.ascontiguousarray(Ls)),
                     _i(np.ascontiguousarray(piv)), _d(X), X.shape[1], X.shape[0])
    return X


def qr_solve(F, T, X, n, b, ib):
    """X <- A^{-1} X = R^{-1} Q^T X with the factors of Algorithm 2."""
    return trsm_upper(F, qr_apply(F, T, X, n, b, ib, trans=True), n, b)


def factor_par(alg: str, tiles: np.ndarray, n: int, b: int, ib: int, nthreads: int):
    """Algorithm 1 / 2 / 3 with the oracle's kernels on a host thread pool (the paper's
    progress-table runtime); bitwise equal to the sequential drivers.
    Returns (aux or None, ipiv or None, info)."""
    p = n // b
    a = {"chol": 0, "qr": 1, "lu": 2}[alg]
    aux = np.zeros(max(1, p * p * ib * b), dtype=np.float64)
    piv = np.zeros(max(1, p * p * b), dtype=np.int32)
    info = lib().o_factor_par(a, n, b, ib, _d(tiles), _d(aux), _i(piv), int(nthreads))
    return (None if a == 0 else aux), (piv if a == 2 else None), info


def lu_decisions(tiles: np.ndarray, n: int, b: int, ib: int):
    """Algorithm 3 as lu(), also returning every pivot decision's (|winner|, |runner-up|)
    in program order (C5 seed-margin instrumentation; the arithmetic is lu()'s)."""
    p = n // b
    cap = p * (p + 1) // 2 * b
    dec = np.zeros(2 * cap, dtype=np.float64)
    lib().o_decisions_arm(_d(dec), cap)
    try:
        Ls, piv, info = lu(tiles, n, b, ib)
        nd = lib().o_decisions_count()
    finally:
        lib().o_decisions_arm(None, 0)
    return Ls, piv, info, dec[:2 * min(nd, cap)].reshape(-1, 2)


def pivot_margin(dec: np.ndarray, dec_perturbed: np.ndarray) -> float:
    """min over decisions of (relative gap between the winner and the
    runner-up) / (relative change of the winner under the input perturbation).  Large
    = the pivot sequence is robust to rounding-level differences; < ~10 = pivot-fragile."""
    best, second = dec[:, 0], dec[:, 1]
    ok = best > 0
    gap = (best[ok] - np.maximum(second[ok], 0.0)) / best[ok]
    chg = np.abs(dec_perturbed[ok, 0] - best[ok]) / best[ok]
    return float(np.min(gap / np.maximum(chg, 2.0 ** -53))) if ok.any() else float("inf")


# ---------------------------------------------------------------- checks

def qr_apply(F, T, X, n, b, ib, trans=False) -> np.ndarray:
    X = np.asfortranarray(X, dtype=np.float64).copy(order="F")
    if X.ndim == 1:
        X = X.reshape(-1, 1, order="F")
    lib().o_qr_apply(n, b, ib, _d(np.ascontiguousarray(F)), _d(np.ascontiguousarray(T)), _d(X),
                     X.shape[1], 1 if trans else 0)
    return X


def lu_apply_N(F, Ls, piv, X, n, b, ib) -> np.ndarray:
    X = np.asfortranarray(X, dtype=np.float64).copy(order="F")
    if X.ndim == 1:
        X = X.reshape(-1, 1, order="F")
    lib().o_lu_apply_N(n, b, ib, _d(np.ascontiguousarray(F)), _d(np.ascontiguousarray(Ls)),
                       _i(np.ascontiguousarray(piv)), _d(X), X.shape[1])
    return X


def chol_residual(A_dense: np.ndarray, L_dense: np.ndarray) -> float:
    n = A_dense.shape[0]
    return lib().o_chol_residual(n, _d(np.asfortranarray(A_dense)), _d(np.asfortranarray(L_dense)))


def ref_chol(A):
    A = np.asfortranarray(A, dtype=np.float64).copy(order="F")
    info = lib().o_ref_chol(A.shape[0], _d(A))
    return A, info


def ref_qr(A):
    A = np.asfortranarray(A, dtype=np.float64).copy(order="F")
    tau = np.zeros(A.shape[0], dtype=np.float64)
    lib().o_ref_qr(A.shape[0], _d(A), _d(tau))
    return A, tau


def ref_gepp(A):
    A = np.asfortranarray(A, dtype=np.float64).copy(order="F")
    piv = np.zeros(A.shape[0], dtype=np.int32)
    info = lib().o_ref_gepp(A.shape[0], _d(A), _i(piv))
    return A, piv, info


def ref_gewp(A):
    A = np.asfortranarray(A, dtype=np.float64).copy(order="F")
    n = A.shape[0]
    sw = np.zeros(n * n, dtype=np.int32)
    info = lib().o_ref_gewp(n, _d(A), _i(sw))
    return A, sw.reshape(n, n, order="F"), info


def kernel_flops(kind: str, b: int, s: int) -> float:
    return lib().o_kernel_flops(KINDS.index(kind), float(b), float(s))


# ---------------------------------------------------------------- dense views of factors

def tile_lower_L(F: np.ndarray, n: int, b: int) -> np.ndarray:
    """Cholesky factor L (dense) from a factored BDL matrix: lower tiles, lower triangle."""
    D = unpack(F, n, n, b)
    return np.tril(D)


def lu_U(F: np.ndarray, n: int, b: int) -> np.ndarray:
    """U of tiled LU (C4): upper triangle of the diagonal tiles and all tiles j > i."""
    D = unpack(F, n, n, b)
    return np.triu(D)


def qr_R(F: np.ndarray, n: int, b: int) -> np.ndarray:
    D = unpack(F, n, n, b)
    return np.triu(D)
