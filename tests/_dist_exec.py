"""CPU executor of the library's multi-GPU plan (test infrastructure).

Each rank (a gloo process) takes its local task graph from ``tile_dist_plan_export`` —
the same host plan the CUDA path uploads — and runs it with the ORACLE's tile kernels on
its own tiles (owner computes on the P x Q block-cyclic grid, include/tilefact.h), in
local program order.  SEND tasks ship the same payload the device SEND items store
into the peers' receive caches (L_kk / L_ik; V_kk copy + T strip; V_ik + T strip; L_kk
copy + ipiv; L_ik + L strip + ipiv) with gloo isend; RECV tasks block on the matching
recv.  The result must be bitwise equal to the sequential oracle (per-tile updates are
chained in k, so any valid distributed order gives the same bits).

This checks the plan's ownership, edges, SEND/RECV pairing and payloads on CPU, with
world_size > 1, without a GPU.
"""
from __future__ import annotations

import numpy as np

import oracle
import tilegen


def _gen(alg, n, seed):
    if alg == "chol":
        return tilegen.spd(n, seed)
    if alg == "qr":
        return tilegen.uniform(n, seed)
    return tilegen.normal(n, seed)


def unit_lower(A):
    X = np.tril(A, -1)
    X[np.diag_indices(A.shape[0])] = 1.0
    return np.asfortranarray(X)


def run_rank(rank, world, alg, n, b, ib, P, Q, seed, port, out_q):
    import os
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = _execute(rank, alg, n, b, ib, P, Q, seed, dist, torch)
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _execute(rank, alg, n, b, ib, P, Q, seed, dist, torch):
    from paper_0709_1272_b200 import tilefact as tf

    p = n // b
    A = _gen(alg, n, seed)
    plan = tf.tile_dist_plan_export(alg, p, P, Q, rank)
    T, S, PV, VX = {}, {}, {}, {}          # owned tiles / strips / pivots / V-L copies
    cT, cS, cP, cV = {}, {}, {}, {}        # receive cache
    for j in range(p):
        for i in range(p):
            if tf.tile_dist_owner(i, j, P, Q) == rank:
                T[(i, j)] = np.asfortranarray(A[i * b:(i + 1) * b, j * b:(j + 1) * b].copy())

    def t(i, j):
        return T[(i, j)] if (i, j) in T else cT[(i, j)]

    def s(i, k):
        return S[(i, k)] if (i, k) in S else cS[(i, k)]

    def pv(i, k):
        return PV[(i, k)] if (i, k) in PV else cP[(i, k)]

    def vx(k):
        return VX[k] if k in VX else cV[k]

    info = 0
    pending = []
    for x in range(len(plan["kind"])):
        kind, k, i, j = (int(plan[c][x]) for c in ("kind", "k", "i", "j"))
        if kind == 0:
            f = oracle.potrf(t(k, k))
            if f and not info:
                info = k * b + f
        elif kind == 1:
            oracle.trsm(t(k, k), t(i, k))
        elif kind == 2:
            oracle.syrk(t(i, k), t(i, i))
        elif kind == 3:
            oracle.gemm_nt(t(i, k), t(j, k), t(i, j))
        elif kind == 4:
            S[(k, k)] = oracle.geqrt(t(k, k), ib)
            VX[k] = unit_lower(t(k, k))
        elif kind == 5:
            oracle.larfb(vx(k), s(k, k), t(k, j), ib)
        elif kind == 6:
            S[(i, k)] = oracle.tsqrt(t(k, k), t(i, k), ib)
        elif kind == 7:
            oracle.ssrfb(t(i, k), s(i, k), t(k, j), t(i, j), ib)
        elif kind == 8:
            PV[(k, k)], f = oracle.getrf(t(k, k), ib)
            VX[k] = unit_lower(t(k, k))
            if f and (not info or k * b + f < info):
                info = k * b + f
        elif kind == 9:
            oracle.gessm(vx(k), pv(k, k), t(k, j), ib)
        elif kind == 10:
            S[(i, k)], PV[(i, k)], f = oracle.tstrf(t(k, k), t(i, k), ib)
            if f and (not info or k * b + f < info):
                info = k * b + f
        elif kind == 11:
            oracle.ssssm(t(i, k), s(i, k), pv(i, k), t(k, j), t(i, j), ib)
        elif kind == 12:   # SEND: the producer's payload to every consumer rank
            parts = _payload(alg, k, i, t, s, pv, vx, producer_is_panel=(i == k))
            buf = torch.from_numpy(np.concatenate([q.ravel(order="F").astype(np.float64) for q in parts]))
            for e in _send_entries(plan, x):
                pending.append(dist.isend(buf.clone(), dst=int(plan["send_peer"][e]), tag=int(plan["gid"][x])))
        elif kind == 13:   # RECV from rank `link`
            src, gid = int(plan["link"][x]), int(plan["gid"][x])
            shapes = _payload_shapes(alg, k, i, b, ib)
            buf = torch.empty(sum(a * c for a, c in shapes), dtype=torch.float64)
            dist.recv(buf, src=src, tag=gid)
            arrs, o = [], 0
            for (a, c) in shapes:
                arrs.append(np.asfortranarray(buf[o:o + a * c].numpy().reshape((a, c), order="F").copy()))
                o += a * c
            _store(alg, k, i, arrs, cT, cS, cP, cV)
    for w in pending:
        w.wait()
    return {"T": {kk: v.copy() for kk, v in T.items()}, "S": {kk: v.copy() for kk, v in S.items()},
            "P": {kk: v.copy() for kk, v in PV.items()}, "info": info,
            "nsend": int((plan["kind"] == 12).sum()), "nrecv": int((plan["kind"] == 13).sum())}


def _send_entries(plan, x):
    """SEND task x's entries: [link, next SEND's link) in send order."""
    kinds = plan["kind"]
    off = int(plan["link"][x])
    nxt = len(plan["send_peer"])
    for y in range(x + 1, len(kinds)):
        if kinds[y] == 12:
            nxt = int(plan["link"][y])
            break
    return range(off, nxt)


def _payload(alg, k, i, t, s, pv, vx, producer_is_panel):
    if alg == "chol":
        return [t(k, k)] if producer_is_panel else [t(i, k)]
    if alg == "qr":
        return [vx(k), s(k, k)] if producer_is_panel else [t(i, k), s(i, k)]
    if producer_is_panel:
        return [vx(k), pv(k, k).reshape(-1, 1)]
    return [t(i, k), s(i, k), pv(i, k).reshape(-1, 1)]


def _payload_shapes(alg, k, i, b, ib):
    panel = i == k
    if alg == "chol":
        return [(b, b)]
    if alg == "qr":
        return [(b, b), (ib, b)]
    return [(b, b), (b, 1)] if panel else [(b, b), (ib, b), (b, 1)]


def _store(alg, k, i, arrs, cT, cS, cP, cV):
    panel = i == k
    if alg == "chol":
        cT[(i, k)] = arrs[0]
        return
    if panel:
        cV[k] = arrs[0]
        if alg == "qr":
            cS[(k, k)] = arrs[1]
        else:
            cP[(k, k)] = arrs[1].ravel().astype(np.int32)
        return
    cT[(i, k)] = arrs[0]
    cS[(i, k)] = arrs[1]
    if alg == "lu":
        cP[(i, k)] = arrs[2].ravel().astype(np.int32)


def sequential(alg, n, b, ib, seed):
    """The sequential oracle on the same input: tiles, strips, pivots, info."""
    A = _gen(alg, n, seed)
    F = oracle.pack(A, b)
    S = piv = None
    info = 0
    if alg == "chol":
        info = oracle.chol(F, n, b)
    elif alg == "qr":
        S = oracle.qr(F, n, b, ib)
    else:
        S, piv, info = oracle.lu(F, n, b, ib)
    return F, S, piv, info
