mkdir -p gpurun_out
./build/kbench gemm 1024 64 1 2 > /dev/null && ncu --set full --clock-control none --import-source on -k regex:kb_kernel -c 1 -o gpurun_out/prof_gemm2 ./build/kbench gemm 1024 64 1 2 > gpurun_out/ncu_gemm2.log 2>&1; echo ncu=$?
