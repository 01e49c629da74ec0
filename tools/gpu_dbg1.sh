K=./build/kbench_wd
for args in "trsm 512 64 1 1" "trsm 256 32 1 1" "potrf 512 64 1 1" "gemm 512 64 1 2" "trsm 128 32 1 1"; do
  echo "== $args"; timeout 60 $K $args 2>&1 | tail -3; echo "rc=$?"
done
