python -c "import oracle; oracle.build()"
for c in 5 4; do
timeout 900 python tools/trace_run.py --config $c --reps 1 --json gpurun_out/trace_c$c.json > /dev/null 2> gpurun_out/trace_c$c.err; echo "trace $c rc=$?"
python -c "import json; d=json.load(open('gpurun_out/trace_c$c.json')); print({k: d[k] for k in ('ms_untraced','busy_frac','mean_gap_us','p50_gap_us')}); print({k:(round(v['mean_us'],1), round(v['gflops_per_sm'],1), round(v['sm_time_share'],3)) for k,v in d['kinds'].items()}); print(d['critical_chain'])"
done
