mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
for a in "ssrfb 512 64 1 2" "ssrfb 256 32 1 4" "ssrfb 128 32 1 8" "gemm 512 64 1 8"; do timeout 60 ./build/kbench $a; done 2>&1 | tee gpurun_out/kb_ssrfb.jsonl
for a in "ssrfb 512 64 1 2" "ssrfb 256 32 1 4"; do timeout 60 ./build/kbench_probe $a; done 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "qr or QR or ssrfb" 2>&1 | tail -3
timeout 600 python bench.py --config 5 --steps 2 --warmup 1 --only --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-300
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --only --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-300
