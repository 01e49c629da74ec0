"""GPU: the device execution trace (the paper's execution-flow view, Fig. fig:flow,
PAPER.md:1014-1026; SPEC.md:360-366 trace validation) checked against the task graph.

With tile_set_trace on, every work item records (task, item, SM, start_ns, end_ns) from
%globaltimer.  For every edge u -> t of the exported DAG (tile_dag_export, or for QR / LU
on the register-slab sizes tile_dag_export_slab: the same graph the scheduler runs), no item of t may start before every item of u has ended, and every
task's items must all be present exactly once.
"""
import numpy as np
import pytest

import tilegen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from _gpu_util import gpu_factor  # noqa: E402
from paper_0709_1272_b200 import tilefact as tf  # noqa: E402


@pytest.mark.parametrize("alg,n,b,ib,slab", [("chol", 1024, 128, 32, 0), ("qr", 1024, 256, 32, 1),
                                             ("lu", 1024, 256, 32, 1), ("qr", 1024, 256, 32, 0),
                                             ("lu", 1024, 256, 32, 0), ("lu", 1536, 512, 64, 1),
                                             ("chol", 2048, 512, 64, 0), ("chol", 2048, 512, 64, 1),
                                             ("chol", 1536, 256, 32, 1)])
def test_trace_respects_dag(alg, n, b, ib, slab):
    A = {"chol": tilegen.spd, "qr": tilegen.uniform, "lu": tilegen.normal}[alg](n, 3)
    tf.tile_set_trace(1 << 22)
    tf.tile_set_slab_dag(slab)
    tf.tile_set_gemm_tile_min(1 if slab else -1)  # panel-level Cholesky: whole-tile GEMM items too
    try:
        gpu_factor(alg, A, b, ib)
        rec = tf.tile_trace_fetch()
        d = tf.tile_dag_export_slab(alg, n // b, b, ib) if slab else tf.tile_dag_export(alg, n // b)
    finally:
        tf.tile_set_trace(0)
        tf.tile_set_slab_dag(-1)
        tf.tile_set_gemm_tile_min(-1)
    nt = len(d["kind"])
    task, item, start, end = rec[:, 0], rec[:, 1], rec[:, 3], rec[:, 4]
    assert len(rec) > 0 and (end >= start).all()
    t_start = np.full(nt, np.iinfo(np.int64).max)
    t_end = np.zeros(nt, dtype=np.int64)
    count = np.zeros(nt, dtype=np.int64)
    np.minimum.at(t_start, task, start)
    np.maximum.at(t_end, task, end)
    np.add.at(count, task, 1)
    assert (count > 0).all(), "every task ran"
    # items of a task are distinct (each popped once)
    pairs = task.astype(np.int64) * 4096 + item
    assert len(np.unique(pairs)) == len(pairs)
    off, succ = d["succ_off"], d["succ"]
    viol = 0
    for u in range(nt):
        for e in range(off[u], off[u + 1]):
            t = succ[e]
            if t_start[t] < t_end[u]:
                viol += 1
    assert viol == 0, f"{viol} edges violated"
