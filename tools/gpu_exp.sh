python -c "import oracle; oracle.build()"
for a in "trsm 512 64 1 2" "trsm 256 32 1 2"; do ./build/kbench $a; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k chol 2>&1 | tail -1
timeout 600 python tools/trace_run.py --config 4 --reps 1 --json gpurun_out/trace_c4.json > /dev/null 2> gpurun_out/trace_c4.err; echo "trace rc=$?"
python -c "import json; d=json.load(open('gpurun_out/trace_c4.json')); print({k: d[k] for k in ('ms_untraced','busy_frac')}); print({k:(round(v['mean_us'],1), round(v['gflops_per_sm'],1)) for k,v in d['kinds'].items()})"
for c in 4 4; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>&1 | tail -1 | cut -c80-200; done
