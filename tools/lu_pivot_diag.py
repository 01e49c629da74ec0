"""Diagnose a GPU-vs-oracle LU pivot mismatch: locate the first differing pivot and print
the oracle's winner / runner-up magnitudes at that decision (near-tie vs bug).
    python tools/lu_pivot_diag.py n b ib seed
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import tilegen  # noqa: E402
from _gpu_util import gpu_factor  # noqa: E402

n, b, ib, seed = (int(x) for x in sys.argv[1:5])
p = n // b
A = tilegen.normal(n, seed)
G, GL, Gp, gi = gpu_factor("lu", A, b, ib)
F = oracle.pack(A, b)
OL, Op, oi, dec = oracle.lu_decisions(F, n, b, ib)
print("info", gi, oi, "pivots equal", np.array_equal(Gp, Op))
d = 0
found = False
for k in range(p):
    for i in range(k, p):
        o = (i + k * p) * b
        g, w = Gp[o:o + b], Op[o:o + b]
        if not np.array_equal(g, w):
            j = int(np.nonzero(g != w)[0][0])
            best, second = dec[d + j]
            print(f"first mismatch: vector ({i},{k}) column {j}: gpu {g[j]} oracle {w[j]}; "
                  f"oracle |winner| {best:.17g} |runner-up| {second:.17g} rel gap {(best - second) / best:.3e}")
            found = True
            break
        d += b
    if found:
        break
r = np.random.default_rng(1234 + seed)
Fp = oracle.pack(A * (1.0 + 2.0 ** -52 * r.standard_normal(A.shape)), b)
_, Pp, _, decp = oracle.lu_decisions(Fp, n, b, ib)
print("perturbed oracle pivots equal oracle:", np.array_equal(Pp, Op))
if np.array_equal(Pp, Op):
    print("margin", oracle.pivot_margin(dec, decp))
