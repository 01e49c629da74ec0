"""ctypes binding of libtilefact.so — same names as the C-ABI in include/tilefact.h.

Argument marshalling only: every step of a factorization runs in the library's CUDA
kernels.  torch is used for device memory and streams.  There is no CPU fallback: if
the shared library is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# TILEFACT_LIB selects another build of the same library (e.g. a TF_CHECK debug build
# from tools/); there is no fallback when it is missing.
LIB_PATH = os.environ.get("TILEFACT_LIB") or os.path.join(_HERE, "libtilefact.so")

KINDS = {"potrf": 0, "trsm": 1, "syrk": 2, "gemm": 3, "geqrt": 4, "larfb": 5, "tsqrt": 6,
         "ssrfb": 7, "getrf": 8, "gessm": 9, "tstrf": 10, "ssssm": 11}
SOLVE_KINDS = {"unitl": 14, "xgessm": 15, "xssssm": 16, "xlarfb": 17, "xssrfb": 18, "xtrsmu": 19, "xgemm": 20,
               "xunssssm": 21, "xungessm": 22}
SLAB_KINDS = {"geqrt_s": 25, "tsqrt_s": 26, "getrf_s": 27, "tstrf_s": 28,  # slab-level DAG panel tasks
              "tsqrt_a": 29, "tstrf_a": 30,  # ... and their off-chain apply tasks
              "potrf_d": 31, "potrf_b": 32, "trsm_p": 33}  # panel-level Cholesky DAG (128-column panels)
KIND_NAMES = {v: k for k, v in KINDS.items()}
KIND_NAMES.update({v: k for k, v in SLAB_KINDS.items()})
ALGS = {"chol": 0, "qr": 1, "lu": 2, "getrs": 3, "ormqr": 4, "qrs": 5, "lu_apply_N": 6}


class TileFactError(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise TileFactError(f"{LIB_PATH} is missing: run `python -m paper_0709_1272_b200.build` "
                            "(there is no fallback path)")
    L = ctypes.CDLL(LIB_PATH)
    i64, i32, vp, sz = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t
    sig = {
        "tile_chol": (i32, [i64, i64, i64, vp, vp, vp]),
        "tile_qr": (i32, [i64, i64, i64, vp, vp, vp]),
        "tile_lu": (i32, [i64, i64, i64, vp, vp, vp, vp, vp]),
        "tile_lu_nopiv": (i32, [i64, i64, i64, vp, vp, vp, vp, vp]),
        "tile_getrs": (i32, [i64, i64, i64, vp, vp, vp, i64, vp, i64, vp]),
        "tile_ormqr": (i32, [i64, i64, i64, vp, vp, i64, vp, i64, vp]),
        "tile_qrs": (i32, [i64, i64, i64, vp, vp, i64, vp, i64, vp]),
        "tile_lu_apply_N": (i32, [i64, i64, i64, vp, vp, vp, i64, vp, i64, vp]),
        "tile_qr_mn": (i32, [i64, i64, i64, i64, vp, vp, vp]),
        "tile_lu_mn": (i32, [i64, i64, i64, i64, vp, vp, vp, vp, vp]),
        "tile_mn_aux_elems": (sz, [i64, i64, i64, i64]),
        "tile_mn_ipiv_elems": (sz, [i64, i64, i64]),
        "tile_qr_t_elems": (sz, [i64, i64, i64]),
        "tile_lu_l_elems": (sz, [i64, i64, i64]),
        "tile_lu_ipiv_elems": (sz, [i64, i64]),
        "tile_pack": (i32, [i64, i64, i64, vp, vp, vp]),
        "tile_unpack": (i32, [i64, i64, i64, vp, vp, vp]),
        "tile_factor_host": (i32, [i32, i64, i64, i64, vp, vp, vp, vp, vp]),
        "tile_set_policy": (None, [i32]),
        "tile_set_slab_dag": (None, [i32]),
        "tile_set_gemm_tile_min": (None, [i32]),
        "tile_set_trace": (None, [i64]),
        "tile_trace_fetch": (i64, [vp, i64]),
        "tile_set_ctas": (None, [i32]),
        "tile_dag_export": (i64, [i32, i64, i32, vp, vp, vp, vp, vp, i64, vp, vp, i64, vp]),
        "tile_dag_export_slab": (i64, [i32, i64, i64, i64, i32, vp, vp, vp, vp, vp, vp, i64, vp, vp, i64, vp]),
        "tk_run": (i32, [i32, i64, i64, vp, vp, vp, vp, vp, vp, vp]),
        "tile_dist_open": (i32, [i32, i64, i64, i64, i32, i32, i32, vp, vp]),
        "tile_dist_ipc_bytes": (i32, []),
        "tile_dist_connect": (i32, [vp, vp]),
        "tile_dist_factor": (i32, [vp, vp, vp, vp, vp, vp]),
        "tile_dist_close": (None, [vp]),
        "tile_dist_probe": (i32, [vp, i32, i32, vp]),
        "tile_dist_probe_read": (i32, [vp, vp]),
        "tile_dist_local_elems": (i64, [i32, i64, i64, i64, i32, i32, i32]),
        "tile_dist_owner": (i32, [i64, i64, i32, i32]),
        "tile_dist_emulate": (i32, [i32, i64, i64, i64, i32, i32, vp, vp, vp, vp, vp]),
        "tile_dist_plan_export": (i64, [i32, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, i64, vp, vp, i64,
                                        vp, vp, i64, vp, vp]),
        "tile_strerror": (ctypes.c_char_p, [i32]),
        "tile_last_error": (ctypes.c_char_p, []),
        "tile_finalize": (None, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()
SYMBOLS = [
    "tile_chol", "tile_qr", "tile_lu", "tile_qr_mn", "tile_lu_mn", "tile_mn_aux_elems", "tile_mn_ipiv_elems",
    "tile_lu_nopiv", "tile_getrs", "tile_ormqr", "tile_qrs", "tile_lu_apply_N",
    "tile_qr_t_elems", "tile_lu_l_elems", "tile_lu_ipiv_elems",
    "tile_pack", "tile_unpack", "tile_factor_host", "tile_set_policy", "tile_set_slab_dag", "tile_set_gemm_tile_min",
    "tile_set_trace",
    "tile_trace_fetch", "tile_set_ctas", "tile_dag_export", "tile_dag_export_slab", "tk_run", "tile_dist_open",
    "tile_dist_ipc_bytes", "tile_dist_connect", "tile_dist_factor", "tile_dist_close",
    "tile_dist_probe", "tile_dist_probe_read",
    "tile_dist_local_elems", "tile_dist_owner", "tile_dist_emulate", "tile_dist_plan_export",
    "tile_strerror", "tile_last_error", "tile_finalize",
]


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _check(rc: int, what: str):
    if rc != 0:
        raise TileFactError(f"{what} failed: rc={rc} ({lib.tile_strerror(rc).decode()}): "
                            f"{lib.tile_last_error().decode()}")


def _dev_f64(t, name, numel=None):
    _dev(t, name, "float64", numel)


def _dev(t, name, dtype, numel=None):
    """The C-ABI takes no buffer lengths: check device, dtype, contiguity and size here so
    an undersized or mistyped tensor is an error, not an out-of-bounds device write."""
    import torch
    want = {"float64": torch.float64, "int32": torch.int32}[dtype]
    if t is None or not (t.is_cuda and t.dtype == want and t.is_contiguous()):
        raise TileFactError(f"{name} must be a contiguous {dtype} CUDA tensor")
    if numel is not None and t.numel() < numel:
        raise TileFactError(f"{name} holds {t.numel()} elements, needs {numel}")


def _info(info):
    if info is not None:
        _dev(info, "info", "int32", 1)


# ------------------------------------------------------------------ factorizations

def tile_chol(n, b, ib, A, info=None, stream=None) -> None:
    """In-place tiled Cholesky of the BDL matrix A (n*n doubles on the device)."""
    _dev_f64(A, "A", n * n)
    _info(info)
    _check(lib.tile_chol(n, b, ib, _ptr(A), _ptr(info), _stream(stream)), "tile_chol")


def tile_qr(n, b, ib, A, T, stream=None) -> None:
    _dev_f64(A, "A", n * n)
    _dev_f64(T, "T", tile_qr_t_elems(n, b, ib))
    _check(lib.tile_qr(n, b, ib, _ptr(A), _ptr(T), _stream(stream)), "tile_qr")


def tile_lu(n, b, ib, A, Ls, ipiv, info=None, stream=None) -> None:
    _dev_f64(A, "A", n * n)
    _dev_f64(Ls, "Ls", tile_lu_l_elems(n, b, ib))
    _dev(ipiv, "ipiv", "int32", tile_lu_ipiv_elems(n, b))
    _info(info)
    _check(lib.tile_lu(n, b, ib, _ptr(A), _ptr(Ls), _ptr(ipiv), _ptr(info), _stream(stream)), "tile_lu")


def tile_lu_nopiv(n, b, ib, A, Ls, ipiv, info=None, stream=None) -> None:
    """GENP in tiled form (Algorithm 3 with every pivot kept)."""
    _dev_f64(A, "A", n * n)
    _dev_f64(Ls, "Ls", tile_lu_l_elems(n, b, ib))
    _dev(ipiv, "ipiv", "int32", tile_lu_ipiv_elems(n, b))
    _info(info)
    _check(lib.tile_lu_nopiv(n, b, ib, _ptr(A), _ptr(Ls), _ptr(ipiv), _ptr(info), _stream(stream)), "tile_lu_nopiv")


def _rhs(X, n):
    """X: CUDA float64 tensor holding a column-major n x nrhs matrix: 1-D (nrhs = 1) or a
    2-D tensor of shape (nrhs, n) (row-major storage of X^T = column-major X)."""
    import torch
    if X.dim() == 1:
        _dev_f64(X, "X", n)
        return 1, n
    if X.dim() != 2 or X.shape[1] != n:
        raise TileFactError("X must be 1-D of length n or 2-D of shape (nrhs, n) (column-major n x nrhs)")
    _dev_f64(X, "X")
    return X.shape[0], n


def tile_getrs(n, b, ib, F, Ls, ipiv, X, stream=None) -> None:
    """X <- A^{-1} X with the tile_lu factors (U^{-1} N^{-1} X, Eq. eq:GETWPcompact)."""
    _dev_f64(F, "F", n * n)
    _dev_f64(Ls, "Ls", tile_lu_l_elems(n, b, ib))
    _dev(ipiv, "ipiv", "int32", tile_lu_ipiv_elems(n, b))
    nrhs, ldx = _rhs(X, n)
    _check(lib.tile_getrs(n, b, ib, _ptr(F), _ptr(Ls), _ptr(ipiv), nrhs, _ptr(X), ldx, _stream(stream)), "tile_getrs")


def tile_lu_apply_N(n, b, ib, F, Ls, ipiv, X, stream=None) -> None:
    """X <- N X (N of Eq. eq:formula N; apply to I for N explicitly)."""
    _dev_f64(F, "F", n * n)
    _dev_f64(Ls, "Ls", tile_lu_l_elems(n, b, ib))
    _dev(ipiv, "ipiv", "int32", tile_lu_ipiv_elems(n, b))
    nrhs, ldx = _rhs(X, n)
    _check(lib.tile_lu_apply_N(n, b, ib, _ptr(F), _ptr(Ls), _ptr(ipiv), nrhs, _ptr(X), ldx, _stream(stream)),
           "tile_lu_apply_N")


def tile_ormqr(n, b, ib, F, T, X, stream=None) -> None:
    """X <- Q^T X with the tile_qr factors."""
    _dev_f64(F, "F", n * n)
    _dev_f64(T, "T", tile_qr_t_elems(n, b, ib))
    nrhs, ldx = _rhs(X, n)
    _check(lib.tile_ormqr(n, b, ib, _ptr(F), _ptr(T), nrhs, _ptr(X), ldx, _stream(stream)), "tile_ormqr")


def tile_qrs(n, b, ib, F, T, X, stream=None) -> None:
    """X <- A^{-1} X = R^{-1} Q^T X with the tile_qr factors."""
    _dev_f64(F, "F", n * n)
    _dev_f64(T, "T", tile_qr_t_elems(n, b, ib))
    nrhs, ldx = _rhs(X, n)
    _check(lib.tile_qrs(n, b, ib, _ptr(F), _ptr(T), nrhs, _ptr(X), ldx, _stream(stream)), "tile_qrs")


def tile_mn_aux_elems(m, n, b, ib) -> int:
    return int(lib.tile_mn_aux_elems(m, n, b, ib))


def tile_mn_ipiv_elems(m, n, b) -> int:
    return int(lib.tile_mn_ipiv_elems(m, n, b))


def tile_qr_mn(m, n, b, ib, A, T, stream=None) -> None:
    """Tiled QR of an m x n BDL matrix (p x q tiles)."""
    _dev_f64(A, "A", m * n)
    _dev_f64(T, "T", tile_mn_aux_elems(m, n, b, ib))
    _check(lib.tile_qr_mn(m, n, b, ib, _ptr(A), _ptr(T), _stream(stream)), "tile_qr_mn")


def tile_lu_mn(m, n, b, ib, A, Ls, ipiv, info=None, stream=None) -> None:
    """Tiled LU with incremental pivoting of an m x n BDL matrix."""
    _dev_f64(A, "A", m * n)
    _dev_f64(Ls, "Ls", tile_mn_aux_elems(m, n, b, ib))
    _dev(ipiv, "ipiv", "int32", tile_mn_ipiv_elems(m, n, b))
    _info(info)
    _check(lib.tile_lu_mn(m, n, b, ib, _ptr(A), _ptr(Ls), _ptr(ipiv), _ptr(info), _stream(stream)), "tile_lu_mn")


def tile_qr_t_elems(n, b, ib) -> int:
    return int(lib.tile_qr_t_elems(n, b, ib))


def tile_lu_l_elems(n, b, ib) -> int:
    return int(lib.tile_lu_l_elems(n, b, ib))


def tile_lu_ipiv_elems(n, b) -> int:
    return int(lib.tile_lu_ipiv_elems(n, b))


def tile_pack(m, n, b, dense, tiles, stream=None) -> None:
    """dense: device float64 holding a column-major m x n matrix (e.g. torch tensor of
    shape (n, m) in row-major = column-major (m, n))."""
    _dev_f64(dense, "dense", m * n)
    _dev_f64(tiles, "tiles", m * n)
    _check(lib.tile_pack(m, n, b, _ptr(dense), _ptr(tiles), _stream(stream)), "tile_pack")


def tile_unpack(m, n, b, tiles, dense, stream=None) -> None:
    _dev_f64(tiles, "tiles", m * n)
    _dev_f64(dense, "dense", m * n)
    _check(lib.tile_unpack(m, n, b, _ptr(tiles), _ptr(dense), _stream(stream)), "tile_unpack")


def tile_factor_host(kind, n, b, ib, hA, hAux=None, hIpiv=None, hInfo=None, stream=None) -> None:
    """End-to-end host-buffer path: hA etc. are CPU tensors (pinned for speed)."""
    k = ALGS[kind] if isinstance(kind, str) else int(kind)
    _check(lib.tile_factor_host(k, n, b, ib, _ptr(hA), _ptr(hAux), _ptr(hIpiv), _ptr(hInfo), _stream(stream)),
           "tile_factor_host")


def tile_set_policy(policy: int) -> None:
    lib.tile_set_policy(int(policy))


def tile_set_slab_dag(on: int) -> None:
    """1 = slab-level QR / LU task graph (default), 0 = tile-level, -1 = default."""
    lib.tile_set_slab_dag(int(on))


def tile_set_gemm_tile_min(min_tiles: int) -> None:
    """Panel-level Cholesky graph: whole-tile GEMM items while a step has >= min_tiles tiles
    outside the lookahead column (0 = strip items everywhere, -1 = default)."""
    lib.tile_set_gemm_tile_min(int(min_tiles))


def tile_set_trace(cap: int) -> None:
    lib.tile_set_trace(int(cap))


def tile_set_ctas(ctas: int) -> None:
    lib.tile_set_ctas(int(ctas))


def tile_trace_fetch(cap: int = 1 << 24):
    """Records of the last factorization: array (N, 5) of task, item, sm, start_ns, end_ns."""
    import numpy as np
    buf = np.zeros((cap, 5), dtype=np.int64)
    got = lib.tile_trace_fetch(ctypes.c_void_p(buf.ctypes.data), cap)
    if got < 0:
        raise TileFactError("tile_trace_fetch failed")
    return buf[:got]


def tile_dag_export(alg, p, policy=1):
    """Host-only: the task graph of Algorithm 1/2/3 for p x p tiles."""
    import numpy as np
    a = ALGS[alg] if isinstance(alg, str) else int(alg)
    ne = ctypes.c_int64(0)
    nt = lib.tile_dag_export(a, p, policy, None, None, None, None, None, 0, None, None, 0, ctypes.byref(ne))
    if nt < 0:
        raise TileFactError("tile_dag_export failed")
    cols = {k: np.zeros(nt, dtype=np.int32) for k in ("kind", "k", "i", "j", "level")}
    off = np.zeros(nt + 1, dtype=np.int64)
    succ = np.zeros(max(1, ne.value), dtype=np.int32)
    P = lambda x: ctypes.c_void_p(x.ctypes.data)  # noqa: E731
    lib.tile_dag_export(a, p, policy, P(cols["kind"]), P(cols["k"]), P(cols["i"]), P(cols["j"]),
                        P(cols["level"]), nt, P(off), P(succ), ne.value, ctypes.byref(ne))
    cols["succ_off"] = off
    cols["succ"] = succ[:ne.value]
    return cols


def tile_dag_export_slab(alg, p, b=128, ib=32, policy=1):
    """Host-only: the slab-level task graph tile_qr / tile_lu run."""
    import numpy as np
    a = ALGS[alg] if isinstance(alg, str) else int(alg)
    ne = ctypes.c_int64(0)
    nt = lib.tile_dag_export_slab(a, p, b, ib, policy, None, None, None, None, None, None, 0, None, None, 0,
                                  ctypes.byref(ne))
    if nt < 0:
        raise TileFactError("tile_dag_export_slab failed")
    cols = {k: np.zeros(nt, dtype=np.int32) for k in ("kind", "k", "i", "j", "slab", "level")}
    off = np.zeros(nt + 1, dtype=np.int64)
    succ = np.zeros(max(1, ne.value), dtype=np.int32)
    P = lambda x: ctypes.c_void_p(x.ctypes.data)  # noqa: E731
    lib.tile_dag_export_slab(a, p, b, ib, policy, P(cols["kind"]), P(cols["k"]), P(cols["i"]), P(cols["j"]),
                             P(cols["slab"]), P(cols["level"]), nt, P(off), P(succ), ne.value, ctypes.byref(ne))
    cols["succ_off"] = off
    cols["succ"] = succ[:ne.value]
    return cols


def tk_run(kind, b, ib, t0=None, t1=None, t2=None, aux=None, ipiv=None, info=None, stream=None) -> None:
    k = KINDS[kind] if isinstance(kind, str) else int(kind)
    _check(lib.tk_run(k, b, ib, _ptr(t0), _ptr(t1), _ptr(t2), _ptr(aux), _ptr(ipiv), _ptr(info), _stream(stream)),
           f"tk_run({kind})")


def tile_finalize() -> None:
    lib.tile_finalize()


# ------------------------------------------------------------------ multi-GPU

def tile_dist_local_elems(alg, n, b, ib, P, Q, which) -> int:
    """Per-rank local buffer sizes: which 0 = A, 1 = T/L strips, 2 = ipiv."""
    a = ALGS[alg] if isinstance(alg, str) else int(alg)
    v = int(lib.tile_dist_local_elems(a, n, b, ib, P, Q, which))
    if v < 0:
        raise TileFactError(f"tile_dist_local_elems: invalid arguments: {lib.tile_last_error().decode()}")
    return v


def tile_dist_owner(i, j, P, Q) -> int:
    return int(lib.tile_dist_owner(i, j, P, Q))


def tile_dist_local_index(i, j, p, P, Q) -> int:
    """Local tile index of global tile (i,j) on its owner (include/tilefact.h layout)."""
    return i // P + (j // Q) * ((p + P - 1) // P)


class DistHandle:
    """One rank of a P x Q multi-GPU factorization (tile_dist_open / connect / factor /
    close).  `exchange(bytes) -> list[bytes]` gathers every rank's IPC handle in rank
    order (e.g. torch.distributed.all_gather_object)."""

    def __init__(self, alg, n, b, ib, P, Q, rank, exchange=None):
        self.alg = ALGS[alg] if isinstance(alg, str) else int(alg)
        self.n, self.b, self.ib, self.P, self.Q, self.rank = n, b, ib, P, Q, rank
        nb = int(lib.tile_dist_ipc_bytes())
        buf = ctypes.create_string_buffer(nb)
        h = ctypes.c_void_p(0)
        _check(lib.tile_dist_open(self.alg, n, b, ib, P, Q, rank, buf, ctypes.byref(h)), "tile_dist_open")
        self._h = h
        if P * Q > 1:
            if exchange is None:
                raise TileFactError("a multi-rank DistHandle needs an `exchange` function")
            allh = exchange(buf.raw)
            if len(allh) != P * Q or any(len(x) != nb for x in allh):
                raise TileFactError("IPC handle exchange returned the wrong shape")
            blob = ctypes.create_string_buffer(b"".join(allh), nb * P * Q)
            _check(lib.tile_dist_connect(self._h, blob), "tile_dist_connect")

    def factor(self, A_loc, aux_loc=None, ipiv_loc=None, info=None, stream=None) -> None:
        args = (self.alg, self.n, self.b, self.ib, self.P, self.Q)
        _dev_f64(A_loc, "A_loc", tile_dist_local_elems(*args, 0))
        if self.alg != 0:
            _dev_f64(aux_loc, "aux_loc", tile_dist_local_elems(*args, 1))
        if self.alg == 2:
            _dev(ipiv_loc, "ipiv_loc", "int32", tile_dist_local_elems(*args, 2))
        _dev(info, "info", "int32", 1)
        _check(lib.tile_dist_factor(self._h, _ptr(A_loc), _ptr(aux_loc), _ptr(ipiv_loc), _ptr(info),
                                    _stream(stream)), "tile_dist_factor")

    def probe(self, peer, value, stream=None) -> None:
        """IPC path check: store `value` into peer's probe slot for this rank (no waiting)."""
        _check(lib.tile_dist_probe(self._h, peer, value, _stream(stream)), "tile_dist_probe")

    def probe_read(self):
        """(slots[8], counter) of this rank's own probe block (synchronizes the device)."""
        import numpy as np
        out = np.zeros(9, dtype=np.int32)
        _check(lib.tile_dist_probe_read(self._h, ctypes.c_void_p(out.ctypes.data)), "tile_dist_probe_read")
        return out[:8], int(out[8])

    def close(self) -> None:
        if self._h:
            lib.tile_dist_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tile_dist_emulate(alg, n, b, ib, P, Q, A_locs, aux_locs=None, ipiv_locs=None, info=None, stream=None) -> None:
    """Run a P x Q job on ONE GPU in one persistent launch (lists of per-rank tensors)."""
    a = ALGS[alg] if isinstance(alg, str) else int(alg)
    R = P * Q

    def arr(ts):
        if ts is None:
            return None
        if len(ts) != R:
            raise TileFactError("need one local buffer per rank")
        return (ctypes.c_void_p * R)(*[t.data_ptr() for t in ts])

    _check(lib.tile_dist_emulate(a, n, b, ib, P, Q, arr(A_locs), arr(aux_locs), arr(ipiv_locs), _ptr(info),
                                 _stream(stream)), "tile_dist_emulate")


def tile_dist_plan_export(alg, p, P, Q, rank):
    """Host-only: rank `rank`'s local task graph (kinds 12 SEND / 13 RECV included)."""
    import numpy as np
    a = ALGS[alg] if isinstance(alg, str) else int(alg)
    ne, ns = ctypes.c_int64(0), ctypes.c_int64(0)
    nt = lib.tile_dist_plan_export(a, p, P, Q, rank, None, None, None, None, None, None, 0, None, None, 0,
                                   None, None, 0, ctypes.byref(ne), ctypes.byref(ns))
    if nt < 0:
        raise TileFactError(f"tile_dist_plan_export failed: {lib.tile_last_error().decode()}")
    cols = {k: np.zeros(nt, dtype=np.int32) for k in ("kind", "k", "i", "j", "link", "gid")}
    off = np.zeros(nt + 1, dtype=np.int64)
    succ = np.zeros(max(1, ne.value), dtype=np.int32)
    sp = np.zeros(max(1, ns.value), dtype=np.int32)
    st = np.zeros(max(1, ns.value), dtype=np.int32)
    P_ = lambda x: ctypes.c_void_p(x.ctypes.data)  # noqa: E731
    lib.tile_dist_plan_export(a, p, P, Q, rank, P_(cols["kind"]), P_(cols["k"]), P_(cols["i"]), P_(cols["j"]),
                              P_(cols["link"]), P_(cols["gid"]), nt, P_(off), P_(succ), ne.value, P_(sp), P_(st),
                              ns.value, ctypes.byref(ne), ctypes.byref(ns))
    cols["succ_off"] = off
    cols["succ"] = succ[:ne.value]
    cols["send_peer"] = sp[:ns.value]
    cols["send_task"] = st[:ns.value]
    return cols


# ------------------------------------------------------------------ flop counts

def lapack_flops(alg: str, n: int) -> float:
    """The paper's GFLOP/s convention: LAPACK counts n^3/3, 4n^3/3, 2n^3/3."""
    return {"chol": n ** 3 / 3.0, "qr": 4.0 * n ** 3 / 3.0, "lu": 2.0 * n ** 3 / 3.0}[alg]


def true_flops(alg: str, n: int, b: int, ib: int) -> float:
    """Leading-order tiled counts: x(1+ib/4b) for QR, x(1+ib/2b) for LU."""
    f = lapack_flops(alg, n)
    if alg == "qr":
        return f * (1 + ib / (4.0 * b))
    if alg == "lu":
        return f * (1 + ib / (2.0 * b))
    return f
