mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
K=./build/kbench
( $K gemm 512 64 1 8; $K syrk 512 64 1 8; $K trsm 512 64 1 4; $K potrf 512 64 1 2;
  $K ssrfb 256 32 1 4; $K ssrfb 512 64 1 2; $K larfb 256 32 1 4; $K tsqrt 256 32 1 2; $K geqrt 256 32 1 2;
  $K ssssm 256 32 1 4; $K gessm 256 32 1 4; $K tstrf 256 32 1 2; $K getrf 256 32 1 2 ) > gpurun_out/kb2.jsonl 2>&1
cat gpurun_out/kb2.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -5
