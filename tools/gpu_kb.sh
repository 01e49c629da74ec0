mkdir -p gpurun_out
K=./build/kbench
( $K gemm 512 64 1 8; $K syrk 512 64 1 8; $K trsm 512 64 1 4; $K potrf 512 64 1 2;
  $K ssrfb 256 32 1 4; $K ssrfb 512 64 1 2; $K larfb 256 32 1 4; $K tsqrt 256 32 1 2; $K geqrt 256 32 1 2;
  $K ssssm 256 32 1 4; $K gessm 256 32 1 4; $K tstrf 256 32 1 2; $K getrf 256 32 1 2; $K tsqrt 512 64 1 1 ) > gpurun_out/kb1.jsonl 2>&1
cat gpurun_out/kb1.jsonl
$K gemm 512 64 1 2 > /dev/null && ncu --set full --clock-control none --import-source on -k regex:kb_kernel -c 1 -o gpurun_out/prof_gemm ./build/kbench gemm 512 64 1 2 > gpurun_out/ncu_gemm.log 2>&1; echo ncu=$?
