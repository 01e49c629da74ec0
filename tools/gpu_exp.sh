python -c "import oracle; oracle.build()"
export TF_DIST_TIMEOUT_S=30
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 600 python tools/trace_run.py --config 4 --json gpurun_out/trace_c4.json > /dev/null 2> gpurun_out/trace_c4.err; echo "trace rc=$?"
python -c "import json; d=json.load(open('gpurun_out/trace_c4.json')); print({k: d[k] for k in ('ms_untraced','busy_frac','mean_gap_us','p50_gap_us')}); print({k:(v['mean_us'], round(v['gflops_per_sm'],1)) for k,v in d['kinds'].items()})"
