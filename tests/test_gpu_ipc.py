"""GPU: the one-process-per-GPU IPC path with two real processes on the one GPU the
test box has, exercised WITHOUT any rank waiting on another.

tile_dist_factor's ranks spin on flags their peers write, and two such ranks as separate
processes on one GPU are not guaranteed to run concurrently (B200_PROFILING.md: Xid 109),
so the factorization itself is covered by the single-launch emulation
(test_gpu_dist.py) and the gloo plan tests (test_dist_host.py).  What this test covers is
everything the emulation cannot: tile_dist_open in two processes, the IPC handle exchange
over torch.distributed (gloo), tile_dist_connect's cudaIpcOpenMemHandle of the peer's
symmetric block, and a device-side system-scope release store plus atomicAdd_system into
the PEER process's memory through that mapping (tile_dist_probe), read back by the peer.
"""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_0709_1272_b200 import tilefact as tf

        def exchange(h):
            out = [None] * world
            dist.all_gather_object(out, h)
            return out

        H = tf.DistHandle("chol", 512, 128, 32, 1, world, rank, exchange=exchange)
        for peer in range(world):
            if peer != rank:
                H.probe(peer, 1000 + 10 * rank + peer)
        torch.cuda.synchronize()
        dist.barrier()
        slots, cnt = H.probe_read()
        dist.barrier()
        H.close()
        dist.destroy_process_group()
        q.put((rank, [int(x) for x in slots], cnt, None))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, None, None, repr(e)))


def test_ipc_probe_two_processes():
    import torch.multiprocessing as mp
    world = 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, slots, cnt, err = q.get(timeout=300)
        assert err is None, f"rank {rank}: {err}"
        res[rank] = (slots, cnt)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        slots, cnt = res[r]
        assert cnt == world - 1
        for peer in range(world):
            want = 1000 + 10 * peer + r if peer != r else 0
            assert slots[peer] == want, (r, peer, slots)
