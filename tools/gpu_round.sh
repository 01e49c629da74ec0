# One gpurun call: GPU parity tests, smoke, the default bench line and optional extras.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tests] [smoke] [bench] [configs] [kb "<kbench args>;..."] [ncu]'
# Each stage writes under gpurun_out/; a stage is skipped unless named.
mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv | tee gpurun_out/smi.txt
export TF_DIST_TIMEOUT_S=30
while [ $# -gt 0 ]; do
  case "$1" in
    tests) timeout 2400 python -m pytest tests -q -m gpu -rA 2>&1 > gpurun_out/pytest_gpu_full.log; echo "pytest rc=$?"
           grep -E "passed|failed|error|\[C5\]|\[config" gpurun_out/pytest_gpu_full.log | tail -40 ;;
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log ;;
    bench) timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
           tail -3 gpurun_out/bench.err; cut -c1-400 gpurun_out/bench.json ;;
    configs) for c in 1 2 3 5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --only --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/bench_c$c.json; cut -c1-200 gpurun_out/bench_c$c.json; done ;;
    kb) shift; IFS=';' read -ra KA <<< "$1"; for a in "${KA[@]}"; do timeout 120 ./build/kbench $a; done 2>&1 | tee -a gpurun_out/kb.jsonl ;;
    ncu) CMD="python bench.py --steps 1 --warmup 1 --only --no-e2e --no-cpu"
         timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
         timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
         timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tf_persistent -s 1 -c 1 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
         ncu -i gpurun_out/prof_c4.ncu-rep --page raw --csv > gpurun_out/prof_c4_raw.csv 2>/dev/null ;;
  esac
  shift
done
