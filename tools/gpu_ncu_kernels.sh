mkdir -p /tmp/ncuk gpurun_out/ncuk
for a in "gemm 512 64 1 2" "ssrfb 512 64 1 1" "tsqrt 512 64 1 1" "geqrt 256 32 1 1" "ssssm 256 32 1 2" "tstrf 256 32 1 1" "getrf 256 32 1 1" "potrf 512 64 1 1" "trsm 512 64 1 1"; do
  set -- $a
  ./build/kbench $a > /tmp/ncuk/plain_$1_$2.log 2>&1 && \
  timeout 300 ncu --set full --clock-control none -k regex:kb_kernel -s 1 -c 1 -o /tmp/ncuk/$1_$2 ./build/kbench $a > /tmp/ncuk/ncu_$1_$2.log 2>&1
  echo "$1 $2 rc=$?"
  ncu -i /tmp/ncuk/$1_$2.ncu-rep --page raw --csv > gpurun_out/ncuk/$1_$2_raw.csv 2>/dev/null
done
ls -la gpurun_out/ncuk
