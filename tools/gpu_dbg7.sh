for args in "t 128 0 7" "t 128 0 0" "t 128 0" "t 512 0" "t 512 -1" "32 96 32 0 128"; do
  echo "== $args"; timeout 30 ./build/dbg_bulk $args 2>&1 | grep -v watchdog | tail -2
done
K=./build/kbench
for a in "gemm 512 64 1 8" "gemm 1024 64 1 4" "syrk 512 64 1 8" "trsm 512 64 1 4" "potrf 512 64 1 2"; do timeout 60 $K $a; done
