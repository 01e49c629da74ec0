# GPU: full parity suite incl. the emulated multi-rank path; quick bench sanity
mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
export TF_DIST_TIMEOUT_S=30
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -30 | tee gpurun_out/pytest_gpu_dist.log
timeout 600 python bench.py --steps 3 --warmup 3 --only --no-e2e --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"
cat gpurun_out/bench_quick.json; tail -3 gpurun_out/bench_quick.err
