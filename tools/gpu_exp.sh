python -c "import oracle; oracle.build()"
for a in "gemm 512 64 1 8" "gemm 256 32 1 8"; do ./build/kbench $a; done
timeout 600 python tools/trace_run.py --config 4 --json gpurun_out/trace_c4.json > /dev/null 2> gpurun_out/trace_c4.err; echo "trace rc=$?"
python -c "import json; d=json.load(open('gpurun_out/trace_c4.json')); print({k: d[k] for k in ('ms_untraced','busy_frac','mean_gap_us','p50_gap_us')}); print({k:(v['mean_us'], round(v['gflops_per_sm'],1)) for k,v in d['kinds'].items()})"
for c in 4 5; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-160; done
export TF_DIST_TIMEOUT_S=30
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x 2>&1 | tail -2
