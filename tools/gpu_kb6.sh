mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
K=./build/kbench
for a in "gemm 512 64 1 8" "trsm 512 64 1 4" "potrf 512 64 1 2"; do timeout 60 $K $a; done 2>&1 | tee gpurun_out/kb6.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench6.json
timeout 300 python tools/trace_run.py --config 4 --json gpurun_out/trace6_c4.json > /dev/null 2>&1
