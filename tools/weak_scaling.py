"""Weak-scaling sweep (the paper's Fig. fig:scal methodology,
PAPER.md:1112-1114: a fixed local size per core, nloc = 5000, as the core count grows).

On one B200 the "cores" of the paper's self-scheduled runtime are the SMs running the
persistent scheduler: the grid is limited to S SMs (tile_set_ctas) and the matrix order
grows as n = nloc * sqrt(S / S0) rounded to a multiple of b, so the memory per SM is fixed
(the paper's convention).  Reported per point: n, S, time, GFLOP/s (LAPACK counts), GFLOP/s
per SM, and efficiency = (GFLOP/s per SM) / (GFLOP/s per SM at the smallest S).  The
multi-GPU form of the same sweep is `bench.py --weak --gpus G` (one rank per GPU).

    python tools/weak_scaling.py [--kinds chol,qr,lu] [--b 256] [--nloc 4096] [--sms 18,37,74,148]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_0709_1272_b200 import tilefact as tf
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", default="chol,qr,lu")
    ap.add_argument("--b", type=int, default=256)
    ap.add_argument("--ib", type=int, default=32)
    ap.add_argument("--nloc", type=int, default=4096, help="matrix order at the smallest SM count")
    ap.add_argument("--sms", default="18,37,74,148")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_weak_scaling.json"))
    args = ap.parse_args()
    sms = [int(x) for x in args.sms.split(",")]
    gen = {"chol": "spd", "qr": "uniform", "lu": "normal"}
    rows = []
    for kind in args.kinds.split(","):
        base = None
        for S in sms:
            n = args.b * max(1, round(args.nloc * math.sqrt(S / sms[0]) / args.b))
            cfg = dict(kind=kind, n=n, b=args.b, ib=args.ib, gen=gen[kind], desc=f"weak {kind} n={n} S={S}")
            tf.tile_set_ctas(S)
            try:
                r, _ = bench.run_device(tf, torch, cfg, args.steps, 2, check=False)
            finally:
                tf.tile_set_ctas(0)
            ms = sum(r["ms"]) / len(r["ms"])
            g = bench.lapack_flops(kind, n) / (ms * 1e-3) / 1e9
            per = g / S
            base = base or per
            row = dict(kind=kind, sms=S, n=n, b=args.b, ib=args.ib, ms=round(ms, 3), gflops=round(g, 1),
                       gflops_per_sm=round(per, 2), efficiency=round(per / base, 3), info=r["info"])
            rows.append(row)
            print(json.dumps(row), flush=True)
    out = {"what": "weak scaling over SMs at fixed memory per SM (n ~ sqrt(SMs)), PAPER.md:1112-1114 methodology",
           "rows": rows}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
