for k in kbench kbench_SKIP_T kbench_SKIP_U kbench_SKIP_W; do echo "$k $(./build/$k ssrfb 512 64 1 2)"; done
./build/kbench ssrfb 256 32 1 4; ./build/kbench ssrfb 128 32 1 8
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "qr or QR or ssrfb" 2>&1 | tail -3
timeout 600 python bench.py --config 5 --steps 2 --warmup 1 --only --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-250
