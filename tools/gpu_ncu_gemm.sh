mkdir -p gpurun_out
./build/kbench gemm 512 64 1 4 > gpurun_out/kb_gemm_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kb_kernel -s 1 -c 1 -o gpurun_out/prof_gemm ./build/kbench gemm 512 64 1 4 > gpurun_out/ncu_gemm.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_gemm.log
