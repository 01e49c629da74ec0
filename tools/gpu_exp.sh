python -c "import oracle; oracle.build()"
for a in "potrf 512 64 1 2" "trsm 512 64 1 2" "potrf 128 32 1 4" "trsm 128 32 1 4"; do ./build/kbench $a; done
for c in 4 1; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>&1 | tail -1 | cut -c80-200; done
export TF_DIST_TIMEOUT_S=30
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x 2>&1 | tail -2
