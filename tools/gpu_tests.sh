python -c "import oracle; oracle.build()"
export TF_DIST_TIMEOUT_S=30
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
for c in 3 2; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/bench_c$c.json; done
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/bench.json
