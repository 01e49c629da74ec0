#!/usr/bin/env python
"""Time the multi-GPU device path on ONE GPU through tile_dist_emulate (P*Q ranks as CTA
groups of one persistent launch): the SEND/RECV protocol overhead relative to the 1-GPU
factorization with the same 148 SMs.  Not a multi-GPU measurement.

    python tools/emu_bench.py --config 4 --grids 1x1,1x2,2x2
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--grids", default="1x1,1x2,2x2")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import torch
    from paper_0709_1272_b200 import tilefact as tf
    cfg = dict(bench.CONFIGS[a.config])
    n, b, ib = cfg["n"], cfg["b"], cfg["ib"]
    p = n // b
    dense = bench.make_dense(cfg, 0, torch.device("cuda"))
    G = torch.empty(n * n, dtype=torch.float64, device="cuda")
    tf.tile_pack(n, n, b, dense.view(-1), G)
    del dense
    torch.cuda.empty_cache()
    out = {"config": cfg["desc"], "grids": {}}
    for gs in a.grids.split(","):
        P, Q = (int(x) for x in gs.split("x"))
        if cfg["kind"] != "chol" and P != 1:
            continue
        R = P * Q
        loc = [tf.tile_dist_local_elems(cfg["kind"], n, b, ib, P, Q, w) for w in range(3)]
        src = {r: [] for r in range(R)}
        for j in range(p):
            for i in range(p):
                src[tf.tile_dist_owner(i, j, P, Q)].append((i + j * p, tf.tile_dist_local_index(i, j, p, P, Q)))
        pristine = []
        bb = b * b
        for r in range(R):
            t = torch.zeros(loc[0], dtype=torch.float64, device="cuda")
            si = torch.tensor([x[0] for x in src[r]], device="cuda")
            di = torch.tensor([x[1] for x in src[r]], device="cuda")
            for c0 in range(0, len(si), 128):
                t.view(-1, bb)[di[c0:c0 + 128]] = G.view(-1, bb)[si[c0:c0 + 128]]
            pristine.append(t)
        work = [torch.empty_like(t) for t in pristine]
        aux = [torch.zeros(loc[1], dtype=torch.float64, device="cuda") for _ in range(R)] if loc[1] else None
        piv = [torch.zeros(loc[2], dtype=torch.int32, device="cuda") for _ in range(R)] if loc[2] else None
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        ms = []
        for rep in range(a.reps + 1):
            for w_, p_ in zip(work, pristine):
                w_.copy_(p_)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            tf.tile_dist_emulate(cfg["kind"], n, b, ib, P, Q, work, aux, piv, info)
            e1.record()
            torch.cuda.synchronize()
            assert int(info.item()) == 0, int(info.item())
            if rep:
                ms.append(e0.elapsed_time(e1))
        m = sum(ms) / len(ms)
        out["grids"][gs] = {"ms": round(m, 2), "tflops": round(bench.lapack_flops(cfg["kind"], n) / (m * 1e-3) / 1e12, 3)}
        del work, pristine, aux, piv
        tf.tile_finalize()
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
