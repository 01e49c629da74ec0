mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
K=./build/kbench
( $K gemm 512 64 1 8; $K gemm 1024 64 1 4; $K syrk 512 64 1 8; $K trsm 512 64 1 4 ) 2>&1 | tee gpurun_out/kb4.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench4.json
