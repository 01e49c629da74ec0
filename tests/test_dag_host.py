"""Host-logic tests of the product's task graph (tile_dag_export; SURVEY §8(a) a13;
PAPER.md:972-1009) and of the C-ABI surface — no GPU needed.

The graph is pinned against (i) closed-form task counts, (ii) an independent generic
RAW/WAR/WAW analysis of the algorithms' read/write sets written here, (iii) the paper's
ready set after the first panel, (iv) the critical-path length 3p-2,
(v) the recursive-subgraph property, and (vi) dependency soundness:
executing the oracle's tile kernels in random topological orders of the exported graph
reproduces the sequential oracle bitwise.
"""
import ctypes
import os
import re

import numpy as np
import pytest
import scipy.linalg

import oracle
import tilegen
from paper_0709_1272_b200 import tilefact as tf

K = tf.KINDS


def _tasks(d):
    return [(int(a), int(b), int(c), int(e)) for a, b, c, e in zip(d["kind"], d["k"], d["i"], d["j"])]


def _preds(d):
    nt = len(d["kind"])
    pr = [set() for _ in range(nt)]
    for t in range(nt):
        for e in range(d["succ_off"][t], d["succ_off"][t + 1]):
            pr[int(d["succ"][e])].add(t)
    return pr


def _rw(alg, kind, k, i, j):
    """Read / write regions of each task (diagonal tiles split into lo / up for QR, LU)."""
    if alg == "chol":
        return {
            K["potrf"]: ([], [("A", k, k)]),
            K["trsm"]: ([("A", k, k)], [("A", i, k)]),
            K["syrk"]: ([("A", i, k)], [("A", i, i)]),
            K["gemm"]: ([("A", i, k), ("A", j, k)], [("A", i, j)]),
        }[kind]
    F, R, C, U = (4, 5, 6, 7) if alg == "qr" else (8, 9, 10, 11)

    def whole(r, c):  # a full tile; diagonal tiles are the union of their two regions
        return [("lo", r, r), ("up", r, r)] if r == c else [("A", r, c)]

    if kind == F:
        return [], whole(k, k) + [("X", k, k)]
    if kind == R:
        return [("lo", k, k), ("X", k, k)], whole(k, j)
    if kind == C:
        return [], [("up", k, k)] + whole(i, k) + [("X", i, k)]
    return whole(i, k) + [("X", i, k)], whole(k, j) + whole(i, j)


def _generic_preds(alg, tasks):
    last_w, readers = {}, {}
    pr = []
    for t, (kind, k, i, j) in enumerate(tasks):
        rd, wr = _rw(alg, kind, k, i, j)
        p = set()
        for r in rd + wr:
            if r in last_w:
                p.add(last_w[r])          # RAW / WAW
        for r in wr:
            p.update(readers.get(r, ()))  # WAR
        p.discard(t)
        for r in rd:
            readers.setdefault(r, set()).add(t)
        for r in wr:
            last_w[r] = t
            readers[r] = set()
        pr.append(p)
    return pr


@pytest.mark.parametrize("alg,p,nt,ne", [("chol", 8, 120, 252), ("qr", 16, 1496, 3960), ("lu", 16, 1496, 3960),
                                         ("qr", 3, 14, None), ("chol", 3, 10, None)])
def test_counts(alg, p, nt, ne):
    d = tf.tile_dag_export(alg, p)
    assert len(d["kind"]) == nt
    if ne is not None:
        assert len(d["succ"]) == ne
    if alg == "chol":
        assert nt == p + p * (p - 1) + p * (p - 1) * (p - 2) // 6
    else:
        assert nt == p + p * (p - 1) + (p - 1) * p * (2 * p - 1) // 6


@pytest.mark.slow
def test_counts_large():
    assert len(tf.tile_dag_export("chol", 64)["succ"]) == 131040
    assert len(tf.tile_dag_export("qr", 64)["succ"]) == 260064


@pytest.mark.parametrize("alg,p", [("chol", 1), ("chol", 5), ("chol", 8), ("qr", 1), ("qr", 4), ("qr", 9),
                                   ("lu", 6)])
def test_matches_generic_dependency_analysis(alg, p):
    d = tf.tile_dag_export(alg, p)
    tasks = _tasks(d)
    assert _preds(d) == _generic_preds(alg, tasks)


def test_ready_set_after_first_panel():
    """SPEC.md:350-351 (0-based): after GEQRT(0) on p = 3: {LARFB(0,1), LARFB(0,2), TSQRT(1,0)}."""
    d = tf.tile_dag_export("qr", 3)
    tasks = _tasks(d)
    pr = _preds(d)
    roots = [t for t in range(len(tasks)) if not pr[t]]
    assert [tasks[t] for t in roots] == [(K["geqrt"], 0, 0, 0)]
    done = {roots[0]}
    ready = {tasks[t] for t in range(len(tasks)) if t not in done and pr[t] <= done}
    assert ready == {(K["larfb"], 0, 0, 1), (K["larfb"], 0, 0, 2), (K["tsqrt"], 0, 1, 0)}


@pytest.mark.parametrize("alg,p", [("chol", 8), ("qr", 16), ("lu", 7), ("chol", 1)])
def test_critical_path(alg, p):
    d = tf.tile_dag_export(alg, p)
    pr = _preds(d)
    depth = [1] * len(pr)
    for t in range(len(pr)):  # program order is a topological order
        if pr[t]:
            depth[t] = 1 + max(depth[x] for x in pr[t])
    assert max(depth) == 3 * p - 2


def test_priorities():
    """GEQRT > TSQRT > LARFB > SSRFB (policy 0 = the paper's ranks)."""
    d = tf.tile_dag_export("qr", 4, policy=0)
    lev = {int(k): set() for k in np.unique(d["kind"])}
    for kind, l in zip(d["kind"], d["level"]):
        lev[int(kind)].add(int(l))
    assert lev[K["geqrt"]] == {0} and lev[K["tsqrt"]] == {1} and lev[K["larfb"]] == {2} and lev[K["ssrfb"]] == {3}
    d = tf.tile_dag_export("chol", 4, policy=0)
    lv = dict(zip(_tasks(d), d["level"]))
    assert lv[(K["potrf"], 1, 1, 1)] < lv[(K["trsm"], 1, 2, 1)] < lv[(K["gemm"], 1, 3, 2)]
    # lookahead policy: updates of the next panel column are promoted
    d = tf.tile_dag_export("chol", 4, policy=1)
    lv = dict(zip(_tasks(d), d["level"]))
    assert lv[(K["gemm"], 0, 3, 1)] < lv[(K["gemm"], 0, 3, 2)]


def test_recursive_subgraph():
    """the DAG for p2 <= p1 is an induced subgraph of the DAG for p1."""
    for alg in ("chol", "qr"):
        small, big = tf.tile_dag_export(alg, 4), tf.tile_dag_export(alg, 7)
        ts, tb = _tasks(small), _tasks(big)
        idx = {t: n for n, t in enumerate(tb)}
        ps, pb = _preds(small), _preds(big)
        for n, t in enumerate(ts):
            assert t in idx
            assert {ts[x] for x in ps[n]} == {tb[x] for x in pb[idx[t]] if tb[x] in set(ts)}


# ------------------------------------------------------------------ dependency soundness

def _run_task(alg, F, X, piv, p, b, ib, task):
    kind, k, i, j = task
    bb = b * b

    def T(r, c):
        return F[(r + c * p) * bb:(r + c * p + 1) * bb].reshape(b, b).T  # view, (row, col)

    def S(r, c):
        o = (r + c * p) * ib * b
        return X[o:o + ib * b].reshape(b, ib).T

    def PV(r, c):
        o = (r + c * p) * b
        return piv[o:o + b]

    def f(a):  # column-major view the oracle can write through
        return np.asfortranarray(a)

    # Each oracle call operates on Fortran views aliasing F / X (T(...) is a transposed
    # view of a C-contiguous block, i.e. a Fortran-contiguous matrix).
    if kind == K["potrf"]:
        oracle.potrf(T(k, k))
    elif kind == K["trsm"]:
        oracle.trsm(T(k, k), T(i, k))
    elif kind == K["syrk"]:
        oracle.syrk(T(i, k), T(i, i))
    elif kind == K["gemm"]:
        oracle.gemm_nt(T(i, k), T(j, k), T(i, j))
    elif kind == K["geqrt"]:
        S(k, k)[:] = oracle.geqrt(T(k, k), ib)
    elif kind == K["larfb"]:
        oracle.larfb(T(k, k), f(S(k, k)), T(k, j), ib)
    elif kind == K["tsqrt"]:
        S(i, k)[:] = oracle.tsqrt(T(k, k), T(i, k), ib)
    elif kind == K["ssrfb"]:
        oracle.ssrfb(T(i, k), f(S(i, k)), T(k, j), T(i, j), ib)
    elif kind == K["getrf"]:
        pv, _ = oracle.getrf(T(k, k), ib)
        PV(k, k)[:] = pv
    elif kind == K["gessm"]:
        oracle.gessm(T(k, k), np.ascontiguousarray(PV(k, k)), T(k, j), ib)
    elif kind == K["tstrf"]:
        ls, pv, _ = oracle.tstrf(T(k, k), T(i, k), ib)
        S(i, k)[:] = ls
        PV(i, k)[:] = pv
    elif kind == K["ssssm"]:
        oracle.ssssm(T(i, k), f(S(i, k)), np.ascontiguousarray(PV(i, k)), T(k, j), T(i, j), ib)


@pytest.mark.parametrize("alg", ["chol", "qr", "lu"])
def test_random_topological_replay_bitwise(alg):
    n, b, ib, p = 48, 12, 4, 4
    A = {"chol": tilegen.spd, "qr": tilegen.uniform, "lu": tilegen.normal}[alg](n, 3)
    ref = oracle.pack(A, b)
    if alg == "chol":
        oracle.chol(ref, n, b)
        refX = None
    elif alg == "qr":
        refX = oracle.qr(ref, n, b, ib)
    else:
        refX, refP, _ = oracle.lu(ref, n, b, ib)
    d = tf.tile_dag_export(alg, p)
    tasks = _tasks(d)
    pr = _preds(d)
    rng = np.random.default_rng(0)
    for rep in range(6):
        F = oracle.pack(A, b)
        X = np.zeros(p * p * ib * b)
        piv = np.zeros(p * p * b, dtype=np.int32)
        indeg = [len(x) for x in pr]
        succ = [[] for _ in tasks]
        for t, ps in enumerate(pr):
            for x in ps:
                succ[x].append(t)
        ready = [t for t in range(len(tasks)) if indeg[t] == 0]
        while ready:
            t = ready.pop(int(rng.integers(len(ready))))
            _run_task(alg, F, X, piv, p, b, ib, tasks[t])
            for s in succ[t]:
                indeg[s] -= 1
                if indeg[s] == 0:
                    ready.append(s)
        assert np.array_equal(F, ref)
        if alg == "qr":
            assert np.array_equal(X, refX)
        if alg == "lu":
            assert np.array_equal(X, refX) and np.array_equal(piv, refP)


# ------------------------------------------------------------------ C-ABI surface

def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "tilefact.h")).read()
    names = set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_0-9]+\s*\*?\s+\**\s*(t[A-Za-z_]+)\s*\(", hdr, re.M))
    assert {"tile_chol", "tile_qr", "tile_lu", "tk_run", "tile_pack"} <= names
    for nm in names:
        assert hasattr(tf.lib, nm), nm
    assert set(tf.SYMBOLS) == names


def test_argument_validation_without_gpu():
    L = tf.lib
    vp = ctypes.c_void_p(16)
    assert L.tile_chol(0, 4, 4, vp, None, None) == -1
    assert L.tile_chol(10, 4, 4, vp, None, None) == -2
    assert L.tile_chol(8, 4, 3, vp, None, None) == -3
    assert L.tile_chol(8, 4, 4, None, None, None) == -4
    assert L.tile_qr(8, 4, 2, vp, None, None) == -5
    assert L.tile_lu(8, 4, 2, vp, vp, None, None, None) == -6
    assert L.tile_qr_t_elems(4096, 256, 32) == 16 * 16 * 32 * 256
    assert L.tile_lu_ipiv_elems(4096, 256) == 16 * 16 * 256
    assert L.tile_strerror(-1) == b"invalid argument"


def test_flop_conventions():
    assert tf.lapack_flops("chol", 32768) == pytest.approx(1.1728e13, rel=1e-4)
    assert tf.lapack_flops("qr", 32768) == pytest.approx(4.6912e13, rel=1e-4)
    assert tf.true_flops("qr", 4096, 256, 32) / tf.lapack_flops("qr", 4096) == pytest.approx(1 + 32 / 1024)


# ------------------------------------------------------------------ solve / apply DAGs (NEXT-3)

def _solve_task(alg, F, S, piv, Xt, p, b, ib, task):
    """One solve-DAG task on the right-hand-side tiles Xt[i] (b x b, Fortran), with the
    oracle's tile kernels for the factorization's own update steps and the textbook
    operations (C4 of SURVEY §8(c)) for the rest."""
    kind, k, i, c = task
    bb = b * b
    T = lambda r, q: F[(r + q * p) * bb:(r + q * p + 1) * bb].reshape(b, b).T  # noqa: E731

    def Sv(r, q):
        o = (r + q * p) * ib * b
        return np.asfortranarray(S[o:o + ib * b].reshape(b, ib).T)

    PV = lambda r, q: np.ascontiguousarray(piv[(r + q * p) * b:(r + q * p + 1) * b])  # noqa: E731
    SK = tf.SOLVE_KINDS
    if kind == SK["unitl"]:
        return
    if kind == SK["xgessm"]:
        oracle.gessm(T(k, k), PV(k, k), Xt[k], ib)
    elif kind == SK["xssssm"]:
        oracle.ssssm(T(i, k), Sv(i, k), PV(i, k), Xt[k], Xt[i], ib)
    elif kind == SK["xlarfb"]:
        oracle.larfb(T(k, k), Sv(k, k), Xt[k], ib)
    elif kind == SK["xssrfb"]:
        oracle.ssrfb(T(i, k), Sv(i, k), Xt[k], Xt[i], ib)
    elif kind == SK["xtrsmu"]:
        Xt[k][:] = scipy.linalg.solve_triangular(np.triu(T(k, k)), Xt[k])
    elif kind == SK["xgemm"]:
        Xt[i][:] = Xt[i] - T(i, k) @ Xt[k]
    elif kind == SK["xunssssm"]:
        L, Ls, pv = T(i, k), Sv(i, k), PV(i, k)
        for s in range(b // ib - 1, -1, -1):
            c0, c1 = s * ib, (s + 1) * ib
            x1 = Xt[k][c0:c1].copy()
            Xt[i][:] = Xt[i] + L[:, c0:c1] @ x1
            Xt[k][c0:c1] = x1 + np.tril(Ls[:, c0:c1], -1) @ x1
            for j in range(c1 - 1, c0 - 1, -1):
                if pv[j] > b:
                    r = pv[j] - b - 1
                    Xt[k][j], Xt[i][r] = Xt[i][r].copy(), Xt[k][j].copy()
    elif kind == SK["xungessm"]:
        Xt[k][:] = Xt[k] + np.tril(T(k, k), -1) @ Xt[k]
        pv = PV(k, k)
        for j in range(b - 1, -1, -1):
            r = pv[j] - 1
            if r != j:
                Xt[k][[j, r]] = Xt[k][[r, j]]


@pytest.mark.parametrize("alg", ["getrs", "ormqr", "qrs", "lu_apply_N"])
def test_solve_dag_random_replay(alg):
    """Dependency soundness of the solve DAGs: random topological orders of the exported
    graph reproduce the program-order result bitwise, and that result is the oracle's
    solve / Q^T / N application (to rounding)."""
    n, b, ib, p = 48, 12, 4, 4
    lu = alg in ("getrs", "lu_apply_N")
    A = (tilegen.normal if lu else tilegen.uniform)(n, 5)
    F = oracle.pack(A, b)
    if lu:
        S, piv, _ = oracle.lu(F, n, b, ib)
    else:
        S, piv = oracle.qr(F, n, b, ib), np.zeros(1, dtype=np.int32)
    Y = np.asfortranarray(tilegen.normal(n, 6)[:, :b])
    d = tf.tile_dag_export(alg, p)
    tasks = _tasks(d)
    pr = _preds(d)
    assert all(t[0] >= 14 for t in tasks)

    def run(order):
        Xt = [np.asfortranarray(Y[r * b:(r + 1) * b].copy()) for r in range(p)]
        for t in order:
            _solve_task(alg, F, S, piv, Xt, p, b, ib, tasks[t])
        return np.vstack(Xt)

    ref = run(range(len(tasks)))
    rng = np.random.default_rng(1)
    for _ in range(4):
        indeg = [len(x) for x in pr]
        succ = [[] for _ in tasks]
        for t, ps in enumerate(pr):
            for x in ps:
                succ[x].append(t)
        ready = [t for t in range(len(tasks)) if indeg[t] == 0]
        order = []
        while ready:
            t = ready.pop(int(rng.integers(len(ready))))
            order.append(t)
            for s_ in succ[t]:
                indeg[s_] -= 1
                if indeg[s_] == 0:
                    ready.append(s_)
        assert len(order) == len(tasks)
        assert np.array_equal(run(order), ref)
    if alg == "getrs":
        want = oracle.lu_solve(F, S, piv, Y, n, b, ib)
    elif alg == "lu_apply_N":
        want = oracle.lu_apply_N(F, S, piv, Y, n, b, ib)
    elif alg == "ormqr":
        want = oracle.qr_apply(F, S, Y, n, b, ib, trans=True)
    else:
        want = oracle.qr_solve(F, S, Y, n, b, ib)
    assert np.max(np.abs(ref - want)) <= 1e-10 * max(1.0, np.max(np.abs(want)))


# ---------------------------------------------------------------- slab-level graph
def _slab_rw(alg, kind, k, i, j, s, S, whole_items, ib=32):
    """Read / write regions of the slab-level tasks, independent of the builder: a tile is
    split into 32-column slabs; a diagonal tile's slab into its upper (rows <= the slab's
    last column) and lower parts; X = T strip / L strip + pivots of a slab, V = the
    explicit V / L copy.  Regions are supersets where a kernel's exact footprint is finer
    (GETRF's interchanges move lower-part rows of every earlier slab; an odd TSTRF slab
    with ib = 64 rewrites rows of the slab before it; GETRF parks state in V)."""
    lu = alg == "lu"
    F, R, C, U = (4, 5, 6, 7) if alg == "qr" else (8, 9, 10, 11)
    FS, CS = (25, 26) if alg == "qr" else (27, 28)
    CA = 29 if alg == "qr" else 30

    def tile(r, c, ss):
        return [("lo", r, r, x) for x in ss] + [("up", r, r, x) for x in ss] if r == c else [("A", r, c, x) for x in ss]

    allS = range(S)
    if kind == FS:
        # left-looking: the earlier slabs' multipliers / reflectors (lower parts, V) and their
        # T / pivots; the upper parts (R / U) of earlier slabs are not read
        rd = [("lo", k, k, x) for x in range(s)] + [("X", k, k, x) for x in range(s)] + \
             [("V", k, x) for x in range(s)]
        wr = [("up", k, k, s), ("lo", k, k, s), ("X", k, k, s)]
        if lu:
            wr += [("lo", k, k, x) for x in range(s)] + [("V", k, x) for x in allS]
        else:
            wr += [("V", k, s)]
        return rd, wr
    if kind == CA:
        # apply task: inner blocks [0, nfull - 1) of TSQRT / TSTRF (i,k) to slab s — reads those
        # blocks' reflectors / multipliers, strips and pivots; rewrites slab s of A_ik and of
        # the diagonal tile's upper part
        nf = (32 * s - (32 * s) % ib) // ib
        last = (nf - 1) * ib // 32  # slabs [0, last) hold blocks 0 .. nf - 2
        rd = [("up", k, k, s)] + [("A", i, k, x) for x in range(last)] + [("X", i, k, x) for x in range(last)]
        return rd, [("up", k, k, s), ("A", i, k, s)]
    if kind == CS:
        prev = [s - 1] if (ib == 64 and s % 2 == 1) else []  # odd slab of a 64-block: L-strip row swaps
        rd = [("up", k, k, s)] + [("A", i, k, x) for x in range(s)] + [("X", i, k, x) for x in range(s)]
        wr = [("up", k, k, s), ("A", i, k, s), ("X", i, k, s)] + [("A", i, k, x) for x in prev] + \
             [("X", i, k, x) for x in prev]
        return rd, wr
    items = allS if whole_items else [s]
    if kind == R:
        return [("V", k, x) for x in allS] + [("X", k, k, x) for x in allS], tile(k, j, items)
    assert kind == U
    return [("A", i, k, x) for x in allS] + [("X", i, k, x) for x in allS], tile(k, j, items) + tile(i, j, items)


@pytest.mark.parametrize("alg,p,b,ib", [("qr", 5, 128, 32), ("lu", 5, 128, 32), ("lu", 4, 256, 32), ("qr", 3, 512, 64),
                                        ("lu", 3, 512, 64), ("qr", 4, 256, 64)])
def test_slab_dag_orders_every_hazard(alg, p, b, ib):
    """Soundness of the slab-level graph: in the builder's program order,
    every read-after-write, write-after-read and write-after-write conflict of the
    independent slab-region model above is ordered by a path of the exported graph; and
    the graph has the expected tasks (panel tasks split per slab, next-column updates per
    slab item)."""
    d = tf.tile_dag_export_slab(alg, p, b, ib)
    S = b // 32
    nt = len(d["kind"])
    F, R, C, U = (4, 5, 6, 7) if alg == "qr" else (8, 9, 10, 11)
    FS, CS = (25, 26) if alg == "qr" else (27, 28)
    kinds = [int(x) for x in d["kind"]]
    # task census
    assert kinds.count(FS) == p * S and kinds.count(CS) == S * p * (p - 1) // 2
    # apply tasks: slabs with >= 2 finished inner blocks before them
    n_ca = sum(1 for s_ in range(S) if (32 * s_ - (32 * s_) % ib) // ib >= 2) * p * (p - 1) // 2
    if alg == "qr":
        n_ca = 0  # only TSTRF is split (tf_sched.h ts_apply_split)
    assert kinds.count(29 if alg == "qr" else 30) == n_ca
    n_split_r = sum(1 for t in range(nt) if kinds[t] == R and d["j"][t] == d["k"][t] + 1)
    assert n_split_r == (p - 1) * S
    pr = _preds(d)
    # whole update tasks: j > k + 1 (one task, S items)
    whole = [kinds[t] in (R, U) and d["j"][t] > d["k"][t] + 1 for t in range(nt)]
    last_w, readers, hazards = {}, {}, []
    for t in range(nt):
        rd, wr = _slab_rw(alg, kinds[t], int(d["k"][t]), int(d["i"][t]), int(d["j"][t]), int(d["slab"][t]), S,
                          whole[t], ib)
        h = set()
        for r in rd + wr:
            if r in last_w:
                h.add(last_w[r])
        for r in wr:
            h.update(readers.get(r, ()))
        h.discard(t)
        hazards.append(h)
        for r in rd:
            readers.setdefault(r, set()).add(t)
        for r in wr:
            last_w[r] = t
            readers[r] = set()
    # ancestors by a forward pass (program order is a topological order of the graph)
    anc = [set() for _ in range(nt)]
    for t in range(nt):
        for u in pr[t]:
            assert u < t, "edges follow program order"
            anc[t] |= anc[u] | {u}
        missing = hazards[t] - anc[t]
        assert not missing, (t, kinds[t], int(d["k"][t]), int(d["i"][t]), int(d["j"][t]), int(d["slab"][t]),
                             [(kinds[u], int(d["k"][u]), int(d["i"][u]), int(d["j"][u]), int(d["slab"][u]))
                              for u in missing])


def test_slab_dag_shorter_chains():
    """The slab-level graph's critical path is much shorter than the tile-level graph's, in
    units of one inner-block application to a 32-column slab (a panel slab = 1, a slab task =
    the blocks it applies + 1, an update item = S): consecutive TSTRF of a column pipeline
    slab by slab and the older blocks of a slab are applied off the chain (PAPER.md:154-159,
    1011-1013)."""
    p, b = 16, 256
    S = b // 32
    d = tf.tile_dag_export_slab("lu", p, b, 32)
    pr = _preds(d)

    def w_fine(t):
        kind, s = int(d["kind"][t]), int(d["slab"][t])
        return {27: s + 1, 28: (1 if s else 0) + 1, 30: s - 1}.get(kind, S)

    L = np.zeros(len(pr))
    for t in range(len(pr)):
        L[t] = w_fine(t) + max((L[u] for u in pr[t]), default=0)
    c = tf.tile_dag_export("lu", p)
    prc = _preds(c)
    Lc = np.zeros(len(prc))
    for t in range(len(prc)):
        w = S * (S + 1) // 2 if int(c["kind"][t]) in (8, 10) else S
        Lc[t] = w + max((Lc[u] for u in prc[t]), default=0)
    assert L.max() < 0.7 * Lc.max(), (L.max(), Lc.max())  # 816 vs 1236 units at p = 16, b = 256


# ---------------------------------------------------------------- panel-level Cholesky graph
def _chol_panel_rw(kind, k, i, j, J, nr):
    """Read / write regions of the panel-level Cholesky tasks, independent of the builder:
    every tile is split into 128 x 128 blocks (tile row, tile col, block row, block col).
    POTRF / TRSM are left-looking over the 128-column panels (PAPER.md:260-274 on blocks):
    panel J of a block row reads that row's and block row J's panels to the left and the
    diagonal block (J,J)."""
    B = lambda r, c, br, bc: (r, c, br, bc)  # noqa: E731
    left = lambda r, c, br: [B(r, c, br, K_) for K_ in range(J)]  # noqa: E731
    if kind == 31:  # diagonal block of panel J
        return left(k, k, J), [B(k, k, J, J)]
    if kind == 32:  # block rows below it
        rd, wr = left(k, k, J) + [B(k, k, J, J)], []
        for r in range(J + 1, nr):
            rd += left(k, k, r)
            wr.append(B(k, k, r, J))
        return rd, wr
    if kind == 33:  # panel J of TRSM (k, i), every block row
        rd, wr = left(k, k, J) + [B(k, k, J, J)], []
        for r in range(nr):
            rd += left(i, k, r)
            wr.append(B(i, k, r, J))
        return rd, wr
    full = lambda r, c: [B(r, c, br, bc) for br in range(nr) for bc in range(nr)]  # noqa: E731
    if kind == 2:  # SYRK writes the lower blocks of (i,i)
        return full(i, k), [B(i, i, br, bc) for br in range(nr) for bc in range(br + 1)]
    assert kind == 3
    return full(i, k) + full(j, k), full(i, j)


@pytest.mark.parametrize("p,b,tile_min", [(5, 256, -1), (4, 384, -1), (4, 512, -1), (3, 1024, -1),
                                          (6, 512, 1), (7, 256, 3), (5, 512, 0), (3, 1280, -1), (3, 1152, 1)])
def test_chol_panel_dag_orders_every_hazard(p, b, tile_min):
    """Soundness of the panel-level Cholesky graph: every RAW / WAR / WAW
    conflict of the independent 128 x 128 block model above is ordered by a path of the
    exported graph, and the graph has the expected task census; also with whole-tile GEMM
    items (tile_set_gemm_tile_min: one item, slab column = 1) in the steps that have at
    least tile_min GEMM tiles outside the lookahead column."""
    tf.tile_set_gemm_tile_min(tile_min)
    try:
        d = tf.tile_dag_export_slab("chol", p, b, 32)
    finally:
        tf.tile_set_gemm_tile_min(-1)
    nr = b // 128
    whole = [t for t in range(len(d["kind"])) if int(d["kind"][t]) == 3 and int(d["slab"][t]) == 1]
    tm = 0 if tile_min < 0 else tile_min  # default: off
    want = sum((p - k - 2) * (p - k - 3) // 2 for k in range(p)
               if tm > 0 and p - k - 1 >= 3 and (p - k - 2) * (p - k - 3) // 2 >= tm)
    assert len(whole) == want
    assert all(int(d["j"][t]) > int(d["k"][t]) + 1 for t in whole)
    nt = len(d["kind"])
    kinds = [int(x) for x in d["kind"]]
    assert kinds.count(31) == p * nr and kinds.count(32) == p * (nr - 1)
    assert kinds.count(33) == nr * p * (p - 1) // 2
    assert kinds.count(2) == p * (p - 1) // 2 and kinds.count(3) == p * (p - 1) * (p - 2) // 6
    assert kinds.count(0) == kinds.count(1) == 0
    pr = _preds(d)
    last_w, readers, hazards = {}, {}, []
    for t in range(nt):
        rd, wr = _chol_panel_rw(kinds[t], int(d["k"][t]), int(d["i"][t]), int(d["j"][t]), int(d["slab"][t]), nr)
        h = set()
        for r in rd + wr:
            if r in last_w:
                h.add(last_w[r])
        for r in wr:
            h.update(readers.get(r, ()))
        h.discard(t)
        hazards.append(h)
        for r in rd:
            readers.setdefault(r, set()).add(t)
        for r in wr:
            last_w[r] = t
            readers[r] = set()
    anc = [set() for _ in range(nt)]
    for t in range(nt):
        for u in pr[t]:
            assert u < t, "edges follow program order"
            anc[t] |= anc[u] | {u}
        missing = hazards[t] - anc[t]
        assert not missing, (t, kinds[t], int(d["k"][t]), int(d["i"][t]), int(d["j"][t]), int(d["slab"][t]),
                             [(kinds[u], int(d["k"][u]), int(d["i"][u]), int(d["j"][u]), int(d["slab"][u]))
                              for u in missing])


def test_chol_panel_dag_shorter_chain():
    """Critical path in units of one 128 x 128 block kernel (a diagonal factorization or a
    triangular solve, with its update): tile-level POTRF = 2 nr - 1 and TRSM = nr units per
    step; panel-level the TRSM panels follow the diagonal blocks one by one, so a step costs
    2 nr - 1 + 1.  SYRK / GEMM items = 1 unit."""
    p, b = 16, 512
    nr = b // 128
    d = tf.tile_dag_export_slab("chol", p, b, 32)
    pr = _preds(d)
    L = np.zeros(len(pr))
    for t in range(len(pr)):
        L[t] = 1 + max((L[u] for u in pr[t]), default=0)
    c = tf.tile_dag_export("chol", p)
    prc = _preds(c)
    Lc = np.zeros(len(prc))
    for t in range(len(prc)):
        w = {0: 2 * nr - 1, 1: nr}.get(int(c["kind"][t]), 1)
        Lc[t] = w + max((Lc[u] for u in prc[t]), default=0)
    assert Lc.max() == (p - 1) * (3 * nr) + 2 * nr - 1
    assert L.max() == (p - 1) * (2 * nr + 1) + 2 * nr - 1
    assert L.max() < 0.8 * Lc.max()
