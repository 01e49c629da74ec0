# LU panel iteration: phase probes (kbench -DTF_PROF_LU) + LU GPU tests + config 3 bench
mkdir -p gpurun_out
python -c "import oracle; oracle.build()" >/dev/null 2>&1
for a in "getrf 256 32" "tstrf 256 32" "getrf 512 64" "tstrf 512 64" "getrf 128 32"; do set -- $a; timeout 60 ./build/kbp_$1 $1 $2 $3 1 4; done 2>&1 | tee gpurun_out/kbp_lu.log
./build/div_check 4; timeout 900 python -m pytest tests -q -m gpu -k "lu or LU or getwp or solve or config3 or div" -x 2>&1 | tail -3
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --only --no-e2e --no-cpu 2>/dev/null | tail -1 | cut -c1-200
