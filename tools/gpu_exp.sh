python -c "import oracle; oracle.build()"
export TF_DIST_TIMEOUT_S=30
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x 2>&1 | tail -2
for c in 2 5; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>&1 | tail -1 | cut -c80-200; done
