for a in "tsqrt 256 32 1 2" "tsqrt 512 64 1 1"; do ./build/kbench_probe $a; done
