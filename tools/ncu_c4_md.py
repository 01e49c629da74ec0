"""Summarise one `ncu --set full` capture of tf_persistent on config 4 (raw CSV page) as
markdown and refresh profiles/ncu_traffic.json.

    python tools/ncu_c4_md.py gpurun_out/prof_c4_<tag>_raw.csv <tag> "<build note>" > profiles/<tag>_ncu_c4.md
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw, tag, note = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(raw)))
d = dict(zip(rows[0], rows[2]))
u = dict(zip(rows[0], rows[1]))
f = lambda k: float(d[k].replace(",", ""))  # noqa: E731
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}
rd = f("dram__bytes_read.sum") * scale[u["dram__bytes_read.sum"]]
wr = f("dram__bytes_write.sum") * scale[u["dram__bytes_write.sum"]]
S = "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio"
print(f"# Round 2 ({note}) — config 4 under ncu\n")
print("`ncu --set full --clock-control none --import-source on -k regex:tf_persistent -s 1 -c 1` of\n"
      "`python bench.py --steps 1 --warmup 1 --only --no-e2e --no-cpu` (tiled Cholesky n = 32768, b = 512,\n"
      "one launch = the whole DAG), after the same command exited 0 without ncu (`tools/gpu_final.sh`;\n"
      f"report `gpurun_out/prof_c4_{tag}.ncu-rep`, not tracked).  Launch list: `profiles/{tag}_launches_c4.csv`.\n")
print("| metric | value |\n|---|---|")
print(f"| gpu__time_duration.sum (cold, serialised) | {f('gpu__time_duration.sum'):.1f} {u['gpu__time_duration.sum']} |")
print(f"| sm__pipe_tensor_subpipe_dmma_cycles_active (pct of peak, active) | **{f('sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active'):.1f} %** |")
print(f"| sm__throughput (pct of peak, elapsed) | {f('sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} % |")
print(f"| smsp__issue_active | {f('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} % |")
print(f"| sm__pipe_fp64_cycles_active (non-tensor FP64) | {f('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.1f} % |")
print(f"| dram__bytes_read.sum | {rd / 1e9:.1f} GB |")
print(f"| dram__bytes_write.sum | {wr / 1e9:.1f} GB |")
print(f"| DRAM traffic per launch (bench `roofline.traffic`) | {(rd + wr) / 1e9:.1f} GB |")
print(f"| lts__t_sector_hit_rate | {f('lts__t_sector_hit_rate.pct'):.1f} % |")
print(f"| registers / thread | {f('launch__registers_per_thread'):.0f} |")
for k in ("math_pipe_throttle", "wait", "long_scoreboard", "short_scoreboard", "barrier", "not_selected", "lg_throttle"):
    print(f"| warps stalled per issue: {k} | {f(S % k):.2f} |")
print("\nAlgorithmic operand traffic of the tiled algorithm (each GEMM reads two 2 MiB tiles and\n"
      "read-modify-writes one): ~p^3/6 x 8 MiB ≈ 350 GB if nothing were reused in L2.  The bound is the\n"
      "FP64 tensor pipe: DMMA active ≈ the bench's fraction of the sustained peak; the top stall is\n"
      "math_pipe_throttle (the DMMA pipe itself), then the fixed-latency wait between dependent issues.")
json.dump({"config4": {"dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
                       "source": f"ncu --set full --clock-control none, tf_persistent, config 4, {note}; "
                                 f"profiles/{tag}_ncu_c4.md"}},
          open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=2)
