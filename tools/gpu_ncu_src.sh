# ncu --set full with source-level sampling for single-kind kbench builds:
#   bash tools/gpu_ncu_src.sh "getrf 256 32" "tsqrt 256 32" ...
mkdir -p gpurun_out
for a in "$@"; do set -- $a
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:kb_kernel -s 1 -c 1 -o gpurun_out/src_$1_$2 ./build/kb_$1 $1 $2 $3 1 2 > gpurun_out/src_$1_$2.log 2>&1; echo "$1 $2 rc=$?"
done
