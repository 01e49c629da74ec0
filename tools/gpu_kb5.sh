mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
K=./build/kbench
for a in "gemm 512 64 1 8" "gemm 1024 64 1 4" "syrk 512 64 1 8" "trsm 512 64 1 4" "potrf 512 64 1 2"; do timeout 60 $K $a; done 2>&1 | tee gpurun_out/kb5.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench5.json
