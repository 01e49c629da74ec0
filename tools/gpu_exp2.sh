for a in "tsqrt 256 32 1 2" "geqrt 256 32 1 2" "tsqrt 512 64 1 1" "geqrt 512 64 1 1"; do ./build/kbench $a; done
