"""CPU baselines for BASELINE.md §5: the oracle (plain C) on configs 1-3 at full size —
sequential drivers (1 thread) and the same kernels on all host cores under the paper's
progress-table runtime — with the CPU model and core count.

    python tools/cpu_baselines.py [--out profiles/r02_cpu_baselines.json] [--configs 1,2,3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    import oracle
    import tilegen
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_cpu_baselines.json"))
    args = ap.parse_args()
    model, ncores = bench.host_cpu()
    rows = []
    for c in (int(x) for x in args.configs.split(",")):
        cfg = bench.CONFIGS[c]
        n, b, ib = cfg["n"], cfg["b"], cfg["ib"]
        A = {"spd": tilegen.spd, "uniform": tilegen.uniform, "normal": tilegen.normal}[cfg["gen"]](n, 0)
        row = {"config": c, "workload": cfg["desc"], "cpu_model": model, "host_cores": ncores}
        for label, nt in (("one_thread", 1), ("all_cores", ncores)):
            F = oracle.pack(A, b)
            t0 = time.perf_counter()
            if nt == 1:
                {"chol": lambda: oracle.chol(F, n, b), "qr": lambda: oracle.qr(F, n, b, ib),
                 "lu": lambda: oracle.lu(F, n, b, ib)}[cfg["kind"]]()
            else:
                oracle.factor_par(cfg["kind"], F, n, b, ib, nt)
            dt = time.perf_counter() - t0
            row[label] = {"s": round(dt, 3), "gflops": round(bench.lapack_flops(cfg["kind"], n) / dt / 1e9, 3),
                          "threads": nt}
        rows.append(row)
        print(json.dumps(row), flush=True)
    json.dump({"what": "oracle CPU baselines (LAPACK flop counts, PAPER.md:1116-1121)", "rows": rows},
              open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
