python -c "import oracle; oracle.build()"
for a in "tsqrt 256 32 1 2" "tsqrt 512 64 1 1" "geqrt 256 32 1 2" "geqrt 512 64 1 1"; do ./build/kbench $a; done
export TF_DIST_TIMEOUT_S=30
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x 2>&1 | tail -4
for c in 2 5 4; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-200; done
