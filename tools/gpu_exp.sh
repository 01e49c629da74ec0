python -c "import oracle; oracle.build()"
for a in "tsqrt 256 32 1 2" "tsqrt 512 64 1 1" "geqrt 256 32 1 2" "geqrt 512 64 1 1" "tsqrt 128 32 1 4"; do ./build/kbench_probe $a; done
export TF_DIST_TIMEOUT_S=30
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x 2>&1 | tail -4
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --only --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-250
timeout 600 python bench.py --config 5 --steps 2 --warmup 1 --only --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-250
