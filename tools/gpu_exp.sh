python -c "import oracle; oracle.build()"
for a in "getrf 256 32 1 2" "tstrf 256 32 1 2" "getrf 512 32 1 1" "tstrf 512 32 1 1" "ssssm 256 32 1 4" "gessm 256 32 1 4"; do ./build/kbench $a; done
export TF_DIST_TIMEOUT_S=30
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x 2>&1 | tail -8
timeout 600 python bench.py --config 3 --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-200
