"""GETWP stability lab (§3.2.4, 804-891) on the GPU.

For 10 seeded N(0,1) matrices of order n = 2048 (the paper's A = randn(n)) and
tile counts p = 1, 2, 4, ..., 128 (b = n/p; p = 1 is GEPP), factor with
tile_lu and report the means of
  * the factorization backward error ||A - N U||_inf / ||A||_inf, both with N U applied
    implicitly (tile_lu_apply_N on U) and — the paper's procedure — with N formed
    explicitly (tile_lu_apply_N on I) and multiplied by U
  * the solution backward error ||y - A x||_inf / (||A||_inf ||x||_inf), x from tile_getrs,
    y a seeded random right-hand side
  * ||N||_inf, ||U||_inf and || |N| |U| ||_inf  (N = tile_lu_apply_N applied to I)
and, for GENP (tile_lu_nopiv, p = 1), the factorization backward error — the paper prints
only two numbers here: mean GENP error 2e-11 vs GETWP p = 128 error 7e-11.
The norms / residual products use torch (measurement harness, not the product path).

    python tools/getwp_lab.py [--n 2048] [--seeds 10] [--pmax 128] [--out profiles/r02_getwp_lab.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def inf_norm(M):
    import torch
    return float(torch.linalg.matrix_norm(M, ord=float("inf")))


def main():
    import numpy as np
    import torch
    import tilegen
    from paper_0709_1272_b200 import tilefact as tf

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--seeds", type=int, default=10)
    ap.add_argument("--pmax", type=int, default=128)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_getwp_lab.json"))
    args = ap.parse_args()
    n = args.n
    dev = torch.device("cuda")
    ps = [p for p in (1, 2, 4, 8, 16, 32, 64, 128, 256) if p <= args.pmax and n % p == 0]
    res = {p: [] for p in ps}
    genp = []
    t0 = time.time()
    for seed in range(args.seeds):
        A_np = tilegen.normal(n, 1000 + seed)                 # column-major numpy
        A = torch.from_numpy(np.ascontiguousarray(A_np.T)).to(dev)   # row-major buffer = A^T; A.t() = A
        At = A.t()
        y = torch.from_numpy(np.random.default_rng(2000 + seed).standard_normal(n)).to(dev)
        nA = inf_norm(At)
        I = torch.eye(n, dtype=torch.float64, device=dev)   # symmetric: its buffer is column-major I
        for p in ps:
            b = n // p
            ib = min(32, b)
            T = torch.empty(n * n, dtype=torch.float64, device=dev)
            tf.tile_pack(n, n, b, A.reshape(-1), T)
            Ls = torch.zeros(tf.tile_lu_l_elems(n, b, ib), dtype=torch.float64, device=dev)
            piv = torch.zeros(tf.tile_lu_ipiv_elems(n, b), dtype=torch.int32, device=dev)
            info = torch.zeros(1, dtype=torch.int32, device=dev)
            tf.tile_lu(n, b, ib, T, Ls, piv, info)
            D = torch.empty(n * n, dtype=torch.float64, device=dev)
            tf.tile_unpack(n, n, b, T, D)
            U = torch.triu(D.view(n, n).t())                 # column-major reading -> U (row-major tensor)
            # N U by the implicit application (columns of U as right-hand sides)
            NU = U.t().contiguous()                           # (n, n) row-major = column-major U
            tf.tile_lu_apply_N(n, b, ib, T, Ls, piv, NU)
            NU = NU.t()
            fact = inf_norm(At - NU) / nA
            # N explicitly (N applied to I)
            N = I.clone()
            tf.tile_lu_apply_N(n, b, ib, T, Ls, piv, N)
            N = N.t()
            # the paper's procedure: N formed explicitly, then N U as a product
            fact_explicit = inf_norm(At - N @ U) / nA
            nN, nU = inf_norm(N), inf_norm(U)
            nNU = inf_norm(N.abs() @ U.abs())
            x = y.clone()
            tf.tile_getrs(n, b, ib, T, Ls, piv, x)
            sol = float((y - At @ x).abs().max()) / (nA * float(x.abs().max()))
            res[p].append(dict(fact=fact, fact_explicit=fact_explicit, sol=sol, N=nN, U=nU, NU=nNU, info=int(info.item())))
            del T, Ls, piv, D, U, NU, N, x
        # GENP: no pivoting at all (b = n)
        T = torch.empty(n * n, dtype=torch.float64, device=dev)
        tf.tile_pack(n, n, n, A.reshape(-1), T)
        Ls = torch.zeros(tf.tile_lu_l_elems(n, n, 32), dtype=torch.float64, device=dev)
        piv = torch.zeros(tf.tile_lu_ipiv_elems(n, n), dtype=torch.int32, device=dev)
        info = torch.zeros(1, dtype=torch.int32, device=dev)
        tf.tile_lu_nopiv(n, n, 32, T, Ls, piv, info)
        D = T.view(n, n).t()                                  # single tile: BDL = column-major
        L = torch.tril(D, -1) + I
        U = torch.triu(D)
        genp.append(dict(fact=inf_norm(At - L @ U) / nA, info=int(info.item())))
        print(f"seed {seed} done ({time.time() - t0:.0f} s)", flush=True)
    mean = lambda v: float(np.mean(v))  # noqa: E731
    out = {
        "what": "GETWP stability on randn(n) (PAPER.md:804-891): means over seeds",
        "n": n, "seeds": args.seeds, "ib": "min(32, b)",
        "getwp": {str(p): {k: mean([r[k] for r in res[p]]) for k in ("fact", "fact_explicit", "sol", "N", "U", "NU")}
                  for p in ps},
        "columns": {"fact": "||A - N U||_inf/||A||_inf with N applied implicitly to U (tile_lu_apply_N)",
                    "fact_explicit": "same with N formed explicitly (N = tile_lu_apply_N(I)) and N U a product, "
                                     "the paper's procedure (P:817-830)",
                    "sol": "||y - A x||_inf / (||A||_inf ||x||_inf), x = tile_getrs(y)",
                    "N": "||N||_inf", "U": "||U||_inf", "NU": "|| |N| |U| ||_inf"},
        "genp": {"fact": mean([g["fact"] for g in genp])},
        "paper": {"genp_fact_mean": 2e-11, "getwp_p128_fact_mean": 7e-11,
                  "source": "PAPER.md:869-871 (MATLAB randn(2048), 10 samples; Opteron)"},
        "infos": sorted({r["info"] for p in ps for r in res[p]} | {g["info"] for g in genp}),
        "seconds": time.time() - t0,
    }
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
