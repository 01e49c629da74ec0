mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
for c in 4 2 3; do timeout 300 python tools/trace_run.py --config $c --json gpurun_out/trace_c$c.json > /dev/null 2> gpurun_out/trace_c$c.err; echo "trace c$c rc=$?"; done
timeout 300 python tools/trace_run.py --config 5 --reps 1 --json gpurun_out/trace_c5.json > /dev/null 2> gpurun_out/trace_c5.err; echo "trace c5 rc=$?"
timeout 300 python tools/trace_run.py --config 4 --n 8192 --reps 1 > gpurun_out/plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tf_persistent -c 1 -o gpurun_out/prof_chol8192 python tools/trace_run.py --config 4 --n 8192 --reps 0 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
