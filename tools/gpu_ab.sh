# A/B on the bench configs (one gpurun call): GPU tests of the task graphs, then each config
# twice.  Environment switches are passed through: TF_FINE=0 (tile-level graphs),
# TF_GEMM_TILE_MIN=<n> (whole-tile GEMM items threshold, 0 = off).
#   bash tools/gpu_ab.sh "<configs>" <steps> ["<env settings to compare>"...]
mkdir -p gpurun_out
python -c "import oracle; oracle.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_slab_dag.py tests/test_gpu_trace.py tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
CFGS="$1"; STEPS="${2:-5}"; shift; shift
[ $# -eq 0 ] && set -- ""
for envs in "$@"; do
  for c in $CFGS; do
    for rep in 1 2; do
      env $envs timeout 900 python bench.py --config $c --steps $STEPS --warmup 3 --only --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/ab_c$c.json
      python - <<PY
import json; d=json.load(open("gpurun_out/ab_c$c.json")); print("[$envs] config $c rep $rep:", d["ms_per_step"], "ms", d["value"], "GFLOP/s", d.get("pct_of_fp64_peak"))
PY
    done
  done
done
