#!/usr/bin/env python
"""Benchmark: FP64 tiled factorizations on B200 (arXiv 0709.1272, BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

A "step" is one whole factorization (every task of Algorithm 1/2/3) of one matrix that
is already resident in HBM, restored from a pristine device copy before each step
(outside the timed region).  The headline workload is BASELINE configs[3] (config 4):
tiled Cholesky FP64, n = 32768, b = 512, SPD A = M M^T/n + n I, M ~ U[-1,1] — the
configuration the north-star target (>= 60% of FP64 tensor peak on 1 B200) is quoted
on.  The other configs are reported in "per_factorization" (3 warm-up + 3 timed steps).
GFLOP/s uses the paper's LAPACK counts n^3/3, 4n^3/3, 2n^3/3.

With N > 1 (torchrun, one rank per GPU) the same n x n factorization is distributed over
a P x Q block-cyclic grid (Cholesky 1x2, 2x2, 2x4; QR/LU 1xN) through tile_dist_factor:
owner-computes, panel tiles stored straight into the consumers' receive caches over
NVLink by the persistent kernel; `value` is the whole job's GFLOP/s (one
factorization per step, max over ranks of the CUDA-event time), "scaling": "strong".

--impl reference times the CPU oracle (oracle/, plain C) on all host cores — its tile
kernels under the paper's progress-table thread pool — on a bounded sample of the same
workload (the reference arm of this tier; there is no reference code).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

CONFIGS = {
    1: dict(kind="chol", n=1024, b=128, ib=32, gen="spd", desc="config1: tiled Cholesky FP64 n=1024 b=128, SPD A=MM^T/n+nI, M~U[-1,1]"),
    2: dict(kind="qr", n=4096, b=256, ib=32, gen="uniform", desc="config2: tiled QR FP64 n=4096 b=256 ib=32, A~U[-0.5,0.5]"),
    3: dict(kind="lu", n=4096, b=256, ib=32, gen="normal", desc="config3: tiled LU (incremental pivoting) FP64 n=4096 b=256 ib=32, A~N(0,1)"),
    4: dict(kind="chol", n=32768, b=512, ib=64, gen="spd", desc="config4: tiled Cholesky FP64 n=32768 b=512, SPD A=MM^T/n+nI, M~U[-1,1]"),
    5: dict(kind="qr", n=32768, b=512, ib=64, gen="uniform", desc="config5: tiled QR FP64 n=32768 b=512 ib=64, A~U[-0.5,0.5]"),
    # the third algorithm at the scale of configs 4-5 (not a BASELINE config)
    6: dict(kind="lu", n=32768, b=512, ib=64, gen="normal", desc="NEXT-1: tiled LU (incremental pivoting) FP64 n=32768 b=512 ib=64, A~N(0,1)"),
}
METRIC = "FP64 GFLOP/s and % of FP64 tensor peak per factorization at 1/2/4/8 B200"
L2_BYTES = 126 * 2**20


def fp64_peak():
    """Measured FP64 DMMA peak (tools/dmma_peak.cu on this pool's B200, profiles/r01_fp64_peak.json);
    MEASURED_PEAKS.json carries no FP64 entry.  Fallback: 148 SM x 128 flop/clk x 1.965 GHz."""
    p = os.path.join(ROOT, "profiles", "r01_fp64_peak.json")
    try:
        d = json.load(open(p))
        return float(d["dmma_tflops_sustained"]), float(max(v for k, v in d.items() if k.startswith("dmma_tflops_t"))), "measured (profiles/r01_fp64_peak.json)"
    except Exception:
        return 37.2, 37.2, "fallback: clock-derived 148*128*1.965e9"


def lapack_flops(kind, n):
    return {"chol": n ** 3 / 3.0, "qr": 4.0 * n ** 3 / 3.0, "lu": 2.0 * n ** 3 / 3.0}[kind]


def true_flops(kind, n, b, ib):
    """Exact per-task sum of the tiled algorithm's flops (leading terms per kernel)."""
    p = n // b
    if kind == "chol":
        return n ** 3 / 3.0 + n ** 2 / 2.0 + n / 6.0
    f = lapack_flops(kind, n)
    return f * (1 + ib / (4.0 * b)) if kind == "qr" else f * (1 + ib / (2.0 * b))


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        load.sort()
        med = load[len(load) // 2] if load else None
        return {"sm_mhz": med, "sm_max_mhz": max(mx) if mx else None, "power_w_max": max(pw) if pw else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------ inputs
def make_dense(cfg, seed, device):
    import tilegen
    n = cfg["n"]
    if cfg["gen"] == "spd":
        return tilegen.spd_torch(n, seed, device)
    if cfg["gen"] == "uniform":
        return tilegen.uniform_torch(n, seed, -0.5, 0.5, device)
    return tilegen.normal_torch(n, seed, device)


def factor(tf, cfg, A, aux, piv, info, stream=None):
    n, b, ib = cfg["n"], cfg["b"], cfg["ib"]
    if cfg["kind"] == "chol":
        tf.tile_chol(n, b, ib, A, info, stream)
    elif cfg["kind"] == "qr":
        tf.tile_qr(n, b, ib, A, aux, stream)
    else:
        tf.tile_lu(n, b, ib, A, aux, piv, info, stream)


def run_device(tf, torch, cfg, steps, warmup, seed=0, want_sample=0, check=True):
    """Times `steps` factorizations (after `warmup`) of a device-resident matrix."""
    dev = torch.device("cuda")
    n, b, ib = cfg["n"], cfg["b"], cfg["ib"]
    dense = make_dense(cfg, seed, dev)
    sample = None
    if want_sample:
        # leading principal block, read column-major (the buffer's transpose = A for SPD)
        import numpy as np
        sample = np.asfortranarray(dense[:want_sample, :want_sample].t().contiguous().cpu().numpy())
    pristine = torch.empty(n * n, dtype=torch.float64, device=dev)
    tf.tile_pack(n, n, b, dense.view(-1), pristine)
    del dense
    work = torch.empty_like(pristine)
    aux = piv = None
    if cfg["kind"] == "qr":
        aux = torch.zeros(tf.tile_qr_t_elems(n, b, ib), dtype=torch.float64, device=dev)
    elif cfg["kind"] == "lu":
        aux = torch.zeros(tf.tile_lu_l_elems(n, b, ib), dtype=torch.float64, device=dev)
        piv = torch.zeros(tf.tile_lu_ipiv_elems(n, b), dtype=torch.int32, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    flush = None
    if n * n * 8 < 2 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES // 8, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for _ in range(warmup):
        work.copy_(pristine)
        factor(tf, cfg, work, aux, piv, info)
    torch.cuda.synchronize()
    for s in range(steps):
        work.copy_(pristine)
        if flush is not None:
            flush.zero_()
        ev[s][0].record(stream)
        factor(tf, cfg, work, aux, piv, info)
        ev[s][1].record(stream)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(bq) for a, bq in ev]
    res = {"ms": ms, "info": int(info.item()), "flush": flush is not None}
    if check:
        res["resid_probe"] = residual_probe(tf, torch, cfg, pristine, work, aux, piv)
    del work, pristine, aux, piv, flush
    torch.cuda.empty_cache()
    return res, sample


def residual_probe(tf, torch, cfg, pristine, F, aux, piv, k=4):
    """||A X - L (L^T X)||_F / (||A||_F ||X||_F) for Cholesky with random probes X
    (plain torch on the unpacked factors — a harness check, not the product path)."""
    if cfg["kind"] != "chol":
        return None
    n, b = cfg["n"], cfg["b"]
    D = torch.empty(n * n, dtype=torch.float64, device="cuda")
    tf.tile_unpack(n, n, b, F, D)
    L = torch.tril(D.view(n, n).t())          # column-major reading -> row-major L
    tf.tile_unpack(n, n, b, pristine, D)
    A = D.view(n, n).t()                       # the full symmetric input
    g = torch.Generator(device="cuda").manual_seed(7)
    X = torch.randn(n, k, dtype=torch.float64, device="cuda", generator=g)
    R = A @ X - L @ (L.t() @ X)
    val = float(torch.linalg.norm(R) / (torch.linalg.norm(A) * torch.linalg.norm(X)))
    del D, L, A, X, R
    torch.cuda.empty_cache()
    return val


def run_e2e(tf, torch, cfg, steps, seed=0):
    """Same metric through tile_factor_host: pinned host BDL buffer -> device -> factor ->
    host; the copies are inside the timed region."""
    n, b, ib = cfg["n"], cfg["b"], cfg["ib"]
    dense = make_dense(cfg, seed, torch.device("cuda"))
    tiles = torch.empty(n * n, dtype=torch.float64, device="cuda")
    tf.tile_pack(n, n, b, dense.view(-1), tiles)
    del dense
    host0 = tiles.cpu()
    del tiles
    torch.cuda.empty_cache()
    hA = torch.empty(n * n, dtype=torch.float64).pin_memory()
    hInfo = torch.zeros(1, dtype=torch.int32)
    hAux = hPiv = None
    if cfg["kind"] != "chol":
        hAux = torch.zeros(tf.tile_qr_t_elems(n, b, ib), dtype=torch.float64).pin_memory()
    if cfg["kind"] == "lu":
        hPiv = torch.zeros(tf.tile_lu_ipiv_elems(n, b), dtype=torch.int32).pin_memory()
    stream = torch.cuda.current_stream()
    ms = []
    for s in range(steps + 1):
        hA.copy_(host0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tf.tile_factor_host(cfg["kind"], n, b, ib, hA, hAux, hPiv, hInfo)
        e1.record(stream)
        torch.cuda.synchronize()
        if s > 0:  # first call allocates the library's device buffers
            ms.append(e0.elapsed_time(e1))
    # bytes the call moves (tile_factor_host streams tile columns: Cholesky only the lower
    # tiles it reads / writes; QR / LU all tiles plus the T / L strips and pivot vectors
    # (i, k), i >= k, that the factorization writes); serial mode (TF_E2E_SERIAL) moves
    # the whole buffers
    p = n // b
    serial = bool(int(os.environ.get("TF_E2E_SERIAL", "0") or 0))
    tiles = p * p if (cfg["kind"] != "chol" or serial) else p * (p + 1) // 2
    strips = p * p if serial else (p * (p + 1) // 2 if cfg["kind"] == "qr" else p * (p - 1) // 2)
    pivs = p * p if serial else p * (p + 1) // 2
    h2d = tiles * b * b * 8
    d2h = tiles * b * b * 8 + (strips * ib * b * 8 if hAux is not None else 0) + \
        (pivs * b * 4 if hPiv is not None else 0) + (4 if cfg["kind"] != "qr" else 0)
    del hA, host0, hAux, hPiv
    return ms, h2d, d2h, int(hInfo.item())


def cpu_oracle_sample(cfg, sample_np, nthreads=1):
    """The oracle as it stands, on the leading principal sample of the same matrix: the
    sequential drivers (nthreads = 1) or the same kernels on the host thread-pool DAG
    executor (the paper's progress-table runtime) with nthreads."""
    import oracle
    ns = sample_np.shape[0]
    b, ib = cfg["b"], cfg["ib"]
    F = oracle.pack(sample_np, b)
    t0 = time.perf_counter()
    if nthreads > 1:
        oracle.factor_par(cfg["kind"], F, ns, b, ib, nthreads)
    elif cfg["kind"] == "chol":
        oracle.chol(F, ns, b)
    elif cfg["kind"] == "qr":
        oracle.qr(F, ns, b, ib)
    else:
        oracle.lu(F, ns, b, ib)
    dt = time.perf_counter() - t0
    return lapack_flops(cfg["kind"], ns) / dt / 1e9, dt


def host_cpu():
    """(CPU model, usable cores) of the host running the CPU baselines."""
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, len(os.sched_getaffinity(0))


def sample_size(cfg):
    # ~10-30 s of single-core oracle work at ~1-2 GFLOP/s, a multiple of b
    target = {"chol": 4096, "qr": 2048, "lu": 2560}[cfg["kind"]]
    ns = max(cfg["b"], (min(target, cfg["n"]) // cfg["b"]) * cfg["b"])
    return ns



# ------------------------------------------------------------------ multi-GPU
def dist_grid(kind, world):
    """P x Q process grid: Cholesky 1x1, 1x2, 2x2, 2x4; QR/LU 1 x G."""
    if kind == "chol":
        return {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}.get(world, (1, world))
    return 1, world


def local_tiles(tf, torch, cfg, G, P, Q, rank):
    """This rank's tiles of the global BDL matrix G, in the library's local layout."""
    n, b, ib = cfg["n"], cfg["b"], cfg["ib"]
    p, bb = n // b, b * b
    src, dst = [], []
    for j in range(p):
        for i in range(p):
            if tf.tile_dist_owner(i, j, P, Q) == rank:
                src.append(i + j * p)
                dst.append(tf.tile_dist_local_index(i, j, p, P, Q))
    loc = torch.zeros(tf.tile_dist_local_elems(cfg["kind"], n, b, ib, P, Q, 0), dtype=torch.float64,
                      device=G.device)
    si = torch.tensor(src, device=G.device)
    di = torch.tensor(dst, device=G.device)
    for c in range(0, len(src), 256):
        loc.view(-1, bb)[di[c:c + 256]] = G.view(-1, bb)[si[c:c + 256]]
    return loc


def run_dist_device(tf, torch, cfg, steps, warmup, rank, world, seed=0):
    """One P x Q factorization per step across `world` GPUs through tile_dist_factor
    (device-initiated panel exchange over NVLink).  Returns per-rank ms list and info."""
    import torch.distributed as dist
    dev = torch.device("cuda")
    n, b, ib = cfg["n"], cfg["b"], cfg["ib"]
    P, Q = dist_grid(cfg["kind"], world)
    dense = make_dense(cfg, seed, dev)
    G = torch.empty(n * n, dtype=torch.float64, device=dev)
    tf.tile_pack(n, n, b, dense.view(-1), G)
    del dense
    pristine = local_tiles(tf, torch, cfg, G, P, Q, rank)
    del G
    torch.cuda.empty_cache()
    work = torch.empty_like(pristine)
    aux = piv = None
    if cfg["kind"] != "chol":
        aux = torch.zeros(tf.tile_dist_local_elems(cfg["kind"], n, b, ib, P, Q, 1), dtype=torch.float64, device=dev)
    if cfg["kind"] == "lu":
        piv = torch.zeros(tf.tile_dist_local_elems(cfg["kind"], n, b, ib, P, Q, 2), dtype=torch.int32, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)

    def exchange(h):
        out = [None] * world
        dist.all_gather_object(out, h)
        return out

    H = tf.DistHandle(cfg["kind"], n, b, ib, P, Q, rank, exchange=exchange)
    stream = torch.cuda.current_stream()
    ms = []
    for s in range(warmup + steps):
        work.copy_(pristine)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        H.factor(work, aux, piv, info)
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        if s >= warmup:
            ms.append(e0.elapsed_time(e1))
        if int(info.item()) != 0:
            raise RuntimeError(f"rank {rank}: tile_dist_factor info={int(info.item())}")
    res = {"ms": ms, "info": int(info.item()), "grid": f"{P}x{Q}"}
    # e2e: host (pinned) local tiles -> device -> factor -> host, copies inside the region
    res["e2e"] = None
    if steps > 0:
        hA = pristine.cpu().pin_memory()
        hOut = torch.empty_like(hA).pin_memory()
        em = []
        for s in range(2):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            work.copy_(hA, non_blocking=True)
            H.factor(work, aux, piv, info)
            hOut.copy_(work, non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            dist.barrier()
            em.append(e0.elapsed_time(e1))
        res["e2e"] = {"ms": sum(em) / len(em), "h2d": hA.numel() * 8, "d2h": hOut.numel() * 8}
        del hA, hOut
    H.close()
    del work, pristine, aux, piv
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------ arms
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import numpy as np
    import tilegen
    cfg = CONFIGS[args.config]
    ns = sample_size(cfg)
    gen = {"spd": lambda: tilegen.spd(ns, 0), "uniform": lambda: tilegen.uniform(ns, 0),
           "normal": lambda: tilegen.normal(ns, 0)}[cfg["gen"]]
    A = gen()
    model, ncores = host_cpu()
    times = []
    for s in range(args.warmup + args.steps):
        g, dt = cpu_oracle_sample(cfg, A, nthreads=ncores)
        if s >= args.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    val = lapack_flops(cfg["kind"], ns) / (ms * 1e-3) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 4), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "n": cfg["n"], "b": cfg["b"], "ib": cfg["ib"],
                   "sample_n": ns, "parallelism": f"{ncores} CPU cores (host thread-pool DAG executor)"},
        "cpu_baseline": {"value": round(val, 4), "unit": "GFLOP/s", "cores": ncores, "kind": "oracle",
                         "cpu_model": model,
                         "sample": f"oracle tile kernels (plain C, -O2) on {ncores} threads of the paper's progress-"
                                   f"table runtime (PAPER.md:1039-1049), {cfg['kind']} on a {ns}x{ns} matrix of the "
                                   f"same recipe (b={cfg['b']}, ib={cfg['ib']}); each step one whole factorization"},
        "e2e": {"value": round(val, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def ncu_traffic(config):
    """DRAM bytes (read + write) per launch of tf_persistent from the committed ncu --set
    full capture of this config (profiles/ncu_traffic.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        e = d.get(f"config{config}")
        return (float(e["dram_bytes_per_launch"]), e["source"]) if e else (None, None)
    except Exception:
        return None, None


def run_ours(args, rank, world, local_rank):
    import torch
    from paper_0709_1272_b200 import build as tfbuild
    if rank == 0:
        tfbuild.build()
    if world > 1:
        torch.distributed.barrier()
    from paper_0709_1272_b200 import tilefact as tf
    torch.cuda.set_device(local_rank)
    cfg = dict(CONFIGS[args.config])
    if args.weak and world > 1:
        cfg["n"] = cfg["b"] * round(cfg["n"] * world ** 0.5 / cfg["b"])
        cfg["desc"] = cfg["desc"] + f" (weak scaling: n scaled by sqrt({world}) to {cfg['n']})"
    n, b, ib = cfg["n"], cfg["b"], cfg["ib"]
    peak_sus, peak_burst, peak_src = fp64_peak()
    launches_per_step = 3  # reset, seed, persistent scheduler kernel (per rank)

    # ---- headline config, device-resident
    clk = ClockSampler(local_rank)
    want = sample_size(cfg) if (rank == 0 and world == 1 and not args.no_cpu) else 0
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk.start()
    sample = None
    if world == 1:
        res, sample = run_device(tf, torch, cfg, args.steps, args.warmup, want_sample=want)
        grid = "1x1"
    else:
        res = run_dist_device(tf, torch, cfg, args.steps, args.warmup, rank, world)
        grid = res["grid"]
    clocks = clk.stop()
    if world > 1:
        torch.distributed.barrier()
    ms_step = sum(res["ms"]) / len(res["ms"])
    if world > 1:
        t = torch.tensor([ms_step], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_step = float(t.item())
    # whole-job throughput: ONE n x n factorization per step, shared by all ranks
    gflops = lapack_flops(cfg["kind"], n) / (ms_step * 1e-3) / 1e9
    tflops_true = true_flops(cfg["kind"], n, b, ib) / (ms_step * 1e-3) / 1e12

    # ---- other factorizations (per-factorization table, 1 GPU only)
    per = []
    if not args.only and rank == 0 and world == 1:
        for c in sorted(CONFIGS):
            if c == args.config or c == 6:  # config 6 (NEXT-1) runs with --config 6
                continue
            cc = CONFIGS[c]
            r, _ = run_device(tf, torch, cc, 3, 3, check=False)
            m = sum(r["ms"]) / len(r["ms"])
            g = lapack_flops(cc["kind"], cc["n"]) / (m * 1e-3) / 1e9
            per.append({"config": c, "workload": cc["desc"], "ms": round(m, 3), "gflops": round(g, 1),
                        "pct_of_fp64_peak": round(100 * g / 1e3 / peak_sus, 2), "info": r["info"],
                        "l2_flushed": r["flush"]})

    # ---- end to end: host buffers, copies inside the timed region
    e2e = None
    if world == 1 and rank == 0 and not args.no_e2e:
        ems, h2d, d2h, einfo = run_e2e(tf, torch, cfg, max(1, min(args.steps, 2)))
        em = sum(ems) / len(ems)
        e2e = {"value": round(lapack_flops(cfg["kind"], n) / (em * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
               "ms_per_step": round(em, 3), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "api": "tile_factor_host (pinned host BDL buffer; tile columns streamed in / out on two copy "
                      "streams, overlapped with the factorization)"
                      if not os.environ.get("TF_E2E_SERIAL") else "tile_factor_host (serial copies)"}
    elif world > 1 and res.get("e2e"):
        t = torch.tensor([res["e2e"]["ms"]], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        em = float(t.item())
        e2e = {"value": round(lapack_flops(cfg["kind"], n) / (em * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
               "ms_per_step": round(em, 3), "h2d_bytes_per_step": res["e2e"]["h2d"] * world,
               "d2h_bytes_per_step": res["e2e"]["d2h"] * world,
               "api": "DistHandle.factor (tile_dist_factor) on each rank's pinned host local tiles"}

    # ---- CPU oracle baseline (bounded sample of the same matrix; rank 0 at N=1 only)
    cpu = None
    if rank == 0 and sample is not None:
        g, dt = cpu_oracle_sample(cfg, sample)
        model, ncores = host_cpu()
        gp, dtp = cpu_oracle_sample(cfg, sample, nthreads=ncores)
        cpu = {"value": round(g, 4), "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
               "sample": f"oracle (plain C, 1 thread) {cfg['kind']} of the leading {sample.shape[0]}x{sample.shape[0]} "
                         f"principal block of the same A, b={b}; {dt:.1f} s",
               "cpu_model": model, "host_cores": ncores,
               "all_cores": {"value": round(gp, 4), "unit": "GFLOP/s", "cores": ncores,
                             "kind": "oracle kernels on a host thread-pool DAG executor (PAPER.md:1039-1049), "
                                     "bitwise equal to the sequential oracle",
                             "seconds": round(dtp, 2)}}

    if rank == 0:
        traffic, tsrc = ncu_traffic(args.config) if world == 1 else (None, None)
        line = {
            "metric": METRIC, "value": round(gflops, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded; BASELINE recipe generated on device)",
            "config": {"workload": cfg["desc"], "n": n, "b": b, "ib": ib, "grid": grid,
                       "parallelism": "1 GPU" if world == 1 else
                       f"{grid} block-cyclic owner-computes, panel tiles over NVLink peer stores",
                       "l2": "inputs (8 GiB) > L2; no flush" if not res.get("flush") else
                       "L2 flushed (256 MiB write) before each step",
                       "policy": "lookahead", "flop_count": "LAPACK n^3/3 (PAPER.md:1116-1121)"},
            "pct_of_fp64_peak": round(100 * gflops / 1e3 / (peak_sus * world), 2),
            "true_tflops": round(tflops_true, 3),
            "roofline": {"bound": "tensor", "kernel": "tf_persistent (one launch = the whole DAG)",
                         "achieved": round(tflops_true / world, 3), "peak": peak_sus, "unit": "TFLOP/s",
                         "frac": round(tflops_true / world / peak_sus, 4),
                         "traffic": traffic, "traffic_source": tsrc,
                         "peak_source": peak_src + "; sustained DMMA figure (kernel runs >0.1 s)",
                         "peak_burst": peak_burst, "per": "GPU" if world > 1 else "launch"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps * world,
            "clocks": clocks,
            "info": res["info"],
            "resid_probe": res.get("resid_probe"),
            "per_factorization": per,
        }
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--only", action="store_true", help="skip the per-factorization table")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: n = n_config * sqrt(N) rounded to a multiple of b (fixed memory per GPU, "
                         "the paper's nloc convention PAPER.md:1112-1114); reports scaling 'weak'")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # launched as `python bench.py --gpus N`: start the N ranks ourselves (one process
        # per GPU, the same torchrun launch the driver uses) and pass the exit code through
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (one rank per GPU)")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    rc = run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
