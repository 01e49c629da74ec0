./build/kbench_probe gemm 512 64 1 8; ./build/kbench_probe gemm 1024 64 1 4; ./build/kbench gemm 512 64 1 8; ./build/kbench gemm 1024 64 1 4
