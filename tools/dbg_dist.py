"""Debug driver: one emulated multi-rank factorization (for compute-sanitizer runs)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
import tilegen
from paper_0709_1272_b200 import tilefact as tf
from test_gpu_dist import run_dist, one_gpu, _gen
from _gpu_util import gpu_pack

alg = sys.argv[1] if len(sys.argv) > 1 else "qr"
n, b, ib, P, Q = [int(x) for x in (sys.argv[2:7] if len(sys.argv) > 6 else (256, 64, 16, 1, 2))]
if len(sys.argv) > 7:
    tf.tile_set_ctas(int(sys.argv[7]))
A = _gen(alg, n, 3)
T0 = gpu_pack(A, b)
R1 = one_gpu(alg, T0.clone(), n, b, ib)
G = run_dist(alg, T0, n, b, ib, P, Q)
print("info", G[3], "equal", torch.equal(G[0], R1[0]) if alg != "chol" else "n/a")
