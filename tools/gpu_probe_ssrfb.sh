for a in "ssrfb 512 64 1 2" "ssrfb 256 32 1 4"; do timeout 60 ./build/kbench_probe $a; done 2>&1
