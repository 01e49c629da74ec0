#!/usr/bin/env python
"""Run one factorization with the device trace on and summarise where the time goes.

    python tools/trace_run.py --config 4 [--n N --b B --ib IB] [--policy 1] [--csv out.csv]

Per task kind: items, mean/max item time, achieved GFLOP/s per SM while running, and
the share of SM-time.  Also: makespan, SM busy fraction, mean gap between consecutive
items on an SM (scheduler overhead), and the critical-path panel chain timing.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def item_flops(kind, b, ib, nitems):
    f = {
        "potrf": b**3 / 3, "trsm": float(b**3), "syrk": b * b * (b + 1.0), "gemm": 2.0 * b**3,
        "geqrt": 4 * b**3 / 3, "larfb": 2.0 * b**3 + 3 * ib * b * b, "tsqrt": 2.0 * b**3 + ib * b * b,
        "ssrfb": 4.0 * b**3 + ib * b * b, "getrf": 2 * b**3 / 3, "gessm": float(b**3),
        "tstrf": b**3 + ib * b * b / 2, "ssssm": 2.0 * b**3 + ib * b * b,
    }[kind]
    return f / nitems


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n", type=int)
    ap.add_argument("--b", type=int)
    ap.add_argument("--ib", type=int)
    ap.add_argument("--policy", type=int, default=1)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--csv")
    ap.add_argument("--json")
    a = ap.parse_args()
    import torch
    from paper_0709_1272_b200 import tilefact as tf
    cfg = dict(bench.CONFIGS[a.config])
    for k in ("n", "b", "ib"):
        if getattr(a, k):
            cfg[k] = getattr(a, k)
    n, b, ib = cfg["n"], cfg["b"], cfg["ib"]
    tf.tile_set_policy(a.policy)
    dense = bench.make_dense(cfg, 0, torch.device("cuda"))
    pristine = torch.empty(n * n, dtype=torch.float64, device="cuda")
    tf.tile_pack(n, n, b, dense.reshape(-1), pristine)
    del dense
    work = torch.empty_like(pristine)
    aux = piv = None
    if cfg["kind"] != "chol":
        aux = torch.zeros(tf.tile_qr_t_elems(n, b, ib), dtype=torch.float64, device="cuda")
    if cfg["kind"] == "lu":
        piv = torch.zeros(tf.tile_lu_ipiv_elems(n, b), dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    # untraced timing
    times = []
    for r in range(a.reps + 1):
        work.copy_(pristine)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bench.factor(tf, cfg, work, aux, piv, info)
        e1.record()
        torch.cuda.synchronize()
        if r:
            times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    tf.tile_set_trace(1 << 30)
    work.copy_(pristine)
    bench.factor(tf, cfg, work, aux, piv, info)
    rec = tf.tile_trace_fetch()
    tf.tile_set_trace(0)
    fine = os.environ.get("TF_FINE", "1") != "0" and (
        (b >= 256 and b % 128 == 0) if cfg["kind"] == "chol" else (b in (128, 256, 512) and ib in (32, 64)))
    d = tf.tile_dag_export_slab(cfg["kind"], n // b, b, ib, a.policy) if fine else tf.tile_dag_export(cfg["kind"], n // b, a.policy)
    kinds = d["kind"][rec[:, 0]]
    t0 = rec[:, 3].min()
    start = (rec[:, 3] - t0) / 1e3
    end = (rec[:, 4] - t0) / 1e3
    dur = end - start
    span = end.max()
    nsm = len(np.unique(rec[:, 2]))
    out = {"config": cfg["desc"], "dag": "slab" if fine else "tile", "n": n, "b": b, "ib": ib, "ms_untraced": ms, "ms_traced_span": span / 1e3,
           "gflops_untraced": bench.lapack_flops(cfg["kind"], n) / (ms * 1e-3) / 1e9,
           "sms": nsm, "items": len(rec), "busy_frac": float(dur.sum() / (nsm * span)), "kinds": {}}
    # gaps between consecutive items on each SM
    gaps = []
    for s in np.unique(rec[:, 2]):
        m = rec[:, 2] == s
        o = np.argsort(start[m])
        st, en = start[m][o], end[m][o]
        if len(st) > 1:
            gaps.extend((st[1:] - en[:-1]).tolist())
    out["mean_gap_us"] = float(np.mean(gaps)) if gaps else 0.0
    out["p50_gap_us"] = float(np.median(gaps)) if gaps else 0.0
    for kid in np.unique(kinds):
        name = tf.KIND_NAMES[int(kid)]
        m = kinds == kid
        nit = int(rec[m, 1].max()) + 1  # items per task of this kind
        if name.endswith("_a"):  # off-chain apply of older inner blocks to one slab
            fl = 0.0
        elif name in ("potrf_d", "potrf_b"):  # one 128 x 128 block of a panel (flops vary with the panel)
            fl = 0.0
        elif name == "trsm_p":  # mean over the panels of a 128-row block
            fl = item_flops("trsm", b, ib, (b // 128) ** 2)
        elif name.endswith("_s"):  # slab-level panel task: one 32-column slab of the tile
            fl = item_flops(name[:-2], b, ib, b // 32)
        else:
            fl = item_flops(name, b, ib, max(nit, b // 32) if name in ("larfb", "ssrfb", "gessm", "ssssm") else nit)
        out["kinds"][name] = {"items": int(m.sum()), "mean_us": float(dur[m].mean()), "max_us": float(dur[m].max()),
                              "gflops_per_sm": float(fl / (dur[m].mean() * 1e-6) / 1e9),
                              "sm_time_share": float(dur[m].sum() / dur.sum())}
    # SM occupancy over time: busy fraction in 20 equal windows of the makespan
    edges = np.linspace(0.0, span, 21)
    occ = []
    for w in range(20):
        lo, hi = edges[w], edges[w + 1]
        occ.append(float(np.clip(np.minimum(end, hi) - np.maximum(start, lo), 0, None).sum() / (nsm * (hi - lo))))
    out["busy_by_window"] = [round(x, 3) for x in occ]
    out["idle_ms_by_window"] = [round((1 - x) * span / 20 / 1e3, 2) for x in occ]
    # the realised critical chain: from the last task to finish, repeatedly step to the
    # predecessor that finished last; time on the chain split into task work and waiting
    tids = rec[:, 0].astype(np.int64)
    nt = len(d["kind"])
    tstart = np.full(nt, np.inf)
    tend = np.zeros(nt)
    np.minimum.at(tstart, tids, start)
    np.maximum.at(tend, tids, end)
    preds = [[] for _ in range(nt)]
    for u in range(nt):
        for e in range(d["succ_off"][u], d["succ_off"][u + 1]):
            preds[int(d["succ"][e])].append(u)
    t = int(np.argmax(tend))
    chain = {"tasks": 0, "work_us": {}, "wait_us": 0.0}
    while True:
        name = tf.KIND_NAMES[int(d["kind"][t])]
        chain["tasks"] += 1
        chain["work_us"][name] = chain["work_us"].get(name, 0.0) + float(tend[t] - tstart[t])
        if not preds[t]:
            chain["wait_us"] += float(tstart[t])
            break
        p = max(preds[t], key=lambda x: tend[x])
        chain["wait_us"] += float(max(0.0, tstart[t] - tend[p]))
        t = p
    chain["work_us"] = {k: round(v, 1) for k, v in chain["work_us"].items()}
    chain["wait_us"] = round(chain["wait_us"], 1)
    out["critical_chain"] = chain
    print(json.dumps(out, indent=1))
    if a.json:
        json.dump(out, open(a.json, "w"), indent=1)
    if a.csv:
        with open(a.csv, "w") as f:
            f.write("sm,kind,k,i,j,item,start_us,end_us\n")
            for r, s_, e_ in zip(rec, start, end):
                t = int(r[0])
                f.write(f"{r[2]},{tf.KIND_NAMES[int(d['kind'][t])]},{d['k'][t]},{d['i'][t]},{d['j'][t]},{r[1]},{s_:.2f},{e_:.2f}\n")


if __name__ == "__main__":
    main()
