mkdir -p gpurun_out
for a in "getrf 256 32" "tstrf 256 32" "geqrt 256 32" "tsqrt 256 32" "potrf 128 32" "potrf 512 64" "getrf 512 64" "tstrf 512 64" "geqrt 512 64" "tsqrt 512 64"; do set -- $a; timeout 60 ./build/kbp_$1 $1 $2 $3 1 4; done 2>&1 | tee gpurun_out/kbp.log
