# Round-2 ncu evidence (one gpurun call):
#  1. per tile kernel: kbench single-kind binaries, one launch each, a focused metric set
#     (DMMA / FP64 pipe activity, issue, DRAM, L2 hit, registers, duration)
#  2. config 4: the bench command exits 0 without ncu, then the launch list, then one
#     --set full capture of tf_persistent (DRAM traffic per launch for the roofline)
mkdir -p gpurun_out/ncuk
M=gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,launch__registers_per_thread,smsp__warps_eligible.avg.per_cycle_active
for a in "gemm 512 64 1 2" "syrk 512 64 1 2" "trsm 512 64 1 2" "trsm 128 32 1 2" "potrf 512 64 1 1" "potrf 128 32 1 2" "ssrfb 512 64 1 1" "ssrfb 256 32 1 2" "tsqrt 512 64 1 1" "tsqrt 256 32 1 1" "geqrt 256 32 1 1" "larfb 256 32 1 2" "ssssm 512 64 1 2" "ssssm 256 32 1 2" "tstrf 256 32 1 1" "getrf 256 32 1 1" "gessm 256 32 1 2"; do
  set -- $a
  ./build/kb_$1 $a > gpurun_out/ncuk/plain_$1_$2.log 2>&1 && \
  timeout 300 ncu --metrics $M --clock-control none -k regex:kb_kernel -s 1 -c 1 --csv ./build/kb_$1 $a > gpurun_out/ncuk/$1_$2.csv 2>&1
  echo "$1 $2 rc=$?"
done
CMD="python bench.py --steps 1 --warmup 1 --only --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_launch_c4.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tf_persistent -s 1 -c 1 -o gpurun_out/prof_c4_${TAG:-r02b} $CMD > gpurun_out/ncu_full_c4.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/prof_c4_${TAG:-r02b}.ncu-rep --page raw --csv > gpurun_out/prof_c4_${TAG:-r02b}_raw.csv 2>/dev/null
