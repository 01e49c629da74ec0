"""Multi-GPU plan, host side, on CPU.

1. Structure: the per-rank local graphs exported by the library (`tile_dist_plan_export`,
   the same plan the CUDA path uploads) partition the global DAG by owner-computes on
   the P x Q block-cyclic grid; every cross-rank edge of the global DAG is exactly one
   SEND (producer rank) -> RECV (consumer rank) pair; no other edges; acyclic.
2. Execution (gloo, world_size 2 and 4): each rank runs its plan with the oracle's tile
   kernels, exchanging the SEND payloads; the union of the ranks' tiles, strips and
   pivots must equal the sequential oracle bitwise (tests/_dist_exec.py).
"""
from __future__ import annotations

import socket
from collections import defaultdict

import numpy as np
import pytest

from paper_0709_1272_b200 import tilefact as tf

GRIDS = [("chol", 1, 1), ("chol", 1, 2), ("chol", 2, 1), ("chol", 2, 2), ("chol", 2, 4),
         ("qr", 1, 2), ("qr", 1, 4), ("qr", 1, 8), ("lu", 1, 2), ("lu", 1, 3)]


def _global(alg, p):
    g = tf.tile_dag_export(alg, p)
    edges = set()
    for u in range(len(g["kind"])):
        for e in range(g["succ_off"][u], g["succ_off"][u + 1]):
            edges.add((u, int(g["succ"][e])))
    return g, edges


def _out_tile(kind, k, i, j):
    if kind in (0, 4, 8):
        return k, k
    if kind in (1, 6, 10):
        return i, k
    if kind in (5, 9):
        return k, j
    if kind == 2:
        return i, i
    return i, j


@pytest.mark.parametrize("alg,P,Q", GRIDS)
@pytest.mark.parametrize("p", [1, 5, 8])
def test_plan_partitions_global_dag(alg, P, Q, p):
    g, gedges = _global(alg, p)
    R = P * Q
    plans = [tf.tile_dist_plan_export(alg, p, P, Q, r) for r in range(R)]
    owner = {}
    for r, pl in enumerate(plans):
        for x in range(len(pl["kind"])):
            kind = int(pl["kind"][x])
            if kind < 12:
                gid = int(pl["gid"][x])
                assert gid not in owner, "task owned twice"
                owner[gid] = r
                assert (kind, int(pl["k"][x]), int(pl["i"][x]), int(pl["j"][x])) == \
                    tuple(int(g[c][gid]) for c in ("kind", "k", "i", "j"))
                ti, tj = _out_tile(kind, int(pl["k"][x]), int(pl["i"][x]), int(pl["j"][x]))
                assert tf.tile_dist_owner(ti, tj, P, Q) == r
    assert sorted(owner) == list(range(len(g["kind"])))
    # reconstruct the global edge set from local edges + SEND/RECV pairs
    got = set()
    recv_src = {}
    for r, pl in enumerate(plans):
        kinds, gids = pl["kind"], pl["gid"]
        for x in range(len(kinds)):
            for e in range(pl["succ_off"][x], pl["succ_off"][x + 1]):
                y = int(pl["succ"][e])
                ky = int(kinds[y])
                assert ky != 13, "RECV tasks have no local predecessors"
                if ky == 12:
                    continue  # producer -> SEND (checked below)
                if kinds[x] == 12:
                    raise AssertionError("SEND tasks have no local successors")
                got.add((int(gids[x]), int(gids[y])))
            if kinds[x] == 13:
                recv_src[(r, int(gids[x]))] = int(pl["link"][x])
                assert int(pl["succ_off"][x + 1] - pl["succ_off"][x]) >= 1
            if kinds[x] == 12:
                # the producer is the SEND's single predecessor, on the same rank
                preds = [u for u in range(len(kinds))
                         for e in range(pl["succ_off"][u], pl["succ_off"][u + 1]) if int(pl["succ"][e]) == x]
                assert len(preds) == 1 and int(gids[preds[0]]) == int(gids[x]) and kinds[preds[0]] < 12
    assert got == gedges
    # every RECV has exactly one SEND entry pointing at it, from the producer's owner
    pointed = defaultdict(int)
    for r, pl in enumerate(plans):
        kinds = pl["kind"]
        for x in range(len(kinds)):
            if kinds[x] != 12:
                continue
            nxt = len(pl["send_peer"])
            for y in range(x + 1, len(kinds)):
                if kinds[y] == 12:
                    nxt = int(pl["link"][y])
                    break
            peers = [int(v) for v in pl["send_peer"][int(pl["link"][x]):nxt]]
            assert len(peers) == len(set(peers)) and r not in peers
            for e in range(int(pl["link"][x]), nxt):
                q, t = int(pl["send_peer"][e]), int(pl["send_task"][e])
                assert int(plans[q]["kind"][t]) == 13 and int(plans[q]["gid"][t]) == int(pl["gid"][x])
                assert int(plans[q]["link"][t]) == r
                pointed[(q, t)] += 1
    for r, pl in enumerate(plans):
        for x in range(len(pl["kind"])):
            if pl["kind"][x] == 13:
                assert pointed[(r, x)] == 1
    if R == 1:
        assert not any(int(k) >= 12 for k in plans[0]["kind"])


@pytest.mark.parametrize("alg,P,Q", [("chol", 2, 2), ("qr", 1, 4), ("lu", 1, 2)])
def test_plan_local_graphs_acyclic(alg, P, Q):
    p = 7
    for r in range(P * Q):
        pl = tf.tile_dist_plan_export(alg, p, P, Q, r)
        n = len(pl["kind"])
        indeg = np.zeros(n, dtype=int)
        for x in range(n):
            for e in range(pl["succ_off"][x], pl["succ_off"][x + 1]):
                indeg[int(pl["succ"][e])] += 1
        ready = [x for x in range(n) if indeg[x] == 0]
        seen = 0
        while ready:
            x = ready.pop()
            seen += 1
            for e in range(pl["succ_off"][x], pl["succ_off"][x + 1]):
                y = int(pl["succ"][e])
                indeg[y] -= 1
                if indeg[y] == 0:
                    ready.append(y)
        assert seen == n


def test_local_buffer_sizes():
    n, b, ib = 4096, 256, 32
    p = n // b
    assert tf.tile_dist_local_elems("chol", n, b, ib, 2, 4, 0) == 8 * 4 * b * b
    assert tf.tile_dist_local_elems("qr", n, b, ib, 1, 4, 1) == p * 4 * ib * b
    assert tf.tile_dist_local_elems("lu", n, b, ib, 1, 3, 2) == p * 6 * b
    assert tf.tile_dist_local_elems("chol", n, b, ib, 1, 1, 0) == n * n
    with pytest.raises(tf.TileFactError):
        tf.tile_dist_local_elems("qr", n, b, ib, 2, 2, 0)  # QR/LU need P = 1
    with pytest.raises(tf.TileFactError):
        tf.tile_dist_local_elems("chol", n, b, ib, 3, 3, 0)  # > 8 ranks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("alg,P,Q,n,b,ib", [
    ("chol", 1, 2, 48, 8, 4),
    ("chol", 2, 2, 56, 8, 4),
    ("qr", 1, 2, 48, 8, 4),
    ("qr", 1, 4, 40, 8, 2),
    ("lu", 1, 2, 48, 8, 4),
])
def test_gloo_plan_execution_matches_sequential_oracle(alg, P, Q, n, b, ib):
    import torch.multiprocessing as mp
    import _dist_exec as de

    R = P * Q
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=de.run_rank, args=(r, R, alg, n, b, ib, P, Q, 3, port, q)) for r in range(R)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(R):
        r, out = q.get(timeout=240)
        res[r] = out
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    F, S, piv, info = de.sequential(alg, n, b, ib, 3)
    p, bb = n // b, b * b
    assert all(res[r]["info"] == 0 for r in res) and info == 0
    if R > 1:
        assert sum(res[r]["nsend"] for r in res) > 0 and sum(res[r]["nrecv"] for r in res) > 0
    for r in range(R):
        for (i, j), T in res[r]["T"].items():
            o = F[(i + j * p) * bb:(i + j * p + 1) * bb].reshape((b, b), order="F")
            if alg == "chol":
                if i < j:
                    continue
                if i == j:
                    T, o = np.tril(T), np.tril(o)
            assert np.array_equal(T, o), (alg, r, i, j)
        for (i, k), Sg in res[r]["S"].items():
            o = S[(i + k * p) * ib * b:(i + k * p + 1) * ib * b].reshape((ib, b), order="F")
            assert np.array_equal(Sg, o), (alg, "strip", i, k)
        for (i, k), pg in res[r]["P"].items():
            assert np.array_equal(pg, piv[(i + k * p) * b:(i + k * p + 1) * b]), (alg, "piv", i, k)
