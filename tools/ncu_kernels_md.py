"""Summarise tools/gpu_ncu_r02.sh output (gpurun_out/ncuk/<kind>_<b>.csv + plain_*.log)
into a markdown table: one row per tile kernel (kbench, one launch of 148 CTAs)."""
import csv, glob, json, os, sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ncuk"
KEYS = [("gpu__time_duration.sum", "ncu duration (us)", 1e-3),
        ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe %", 1),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %", 1),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %", 1),
        ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps/cyc", 1),
        ("dram__bytes_read.sum", "DRAM rd (MB)", 1e-6),
        ("dram__bytes_write.sum", "DRAM wr (MB)", 1e-6),
        ("lts__t_sector_hit_rate.pct", "L2 hit %", 1),
        ("launch__registers_per_thread", "regs", 1)]
rows = []
for f in sorted(glob.glob(os.path.join(src, "*_*.csv"))):
    base = os.path.basename(f)[:-4]
    if base.endswith("_raw"):
        continue
    kind, b = base.rsplit("_", 1)
    m = {}
    for line in open(f):
        if not line.startswith('"0"'):
            continue
        r = next(csv.reader([line]))
        m[r[-3]] = float(r[-1].replace(",", ""))
    plain = os.path.join(src, f"plain_{kind}_{b}.log")
    kb = None
    if os.path.exists(plain):
        for line in open(plain):
            if line.startswith("{"):
                kb = json.loads(line)
    rows.append((kind, int(b), m, kb))
print("| kernel (kbench, b) | us/item (no ncu) | GF/s/SM (no ncu) | " + " | ".join(k[1] for k in KEYS) + " |")
print("|---" * (3 + len(KEYS)) + "|")
for kind, b, m, kb in rows:
    cells = [f"{kind} b={b}", f"{kb['us_per_item']:.1f}" if kb else "-", f"{kb['gflops_per_sm']:.1f}" if kb else "-"]
    for k, _, s in KEYS:
        cells.append(f"{m[k] * s:.1f}" if k in m else "-")
    print("| " + " | ".join(cells) + " |")
