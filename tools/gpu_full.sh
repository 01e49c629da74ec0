# one GPU call: parity tests, default bench, launch list, one ncu --set full of the top kernel
mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
export TF_DIST_TIMEOUT_S=30
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
CMD="python bench.py --steps 1 --warmup 1 --only --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tf_persistent -s 1 -c 1 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
ncu -i gpurun_out/prof_c4.ncu-rep --page raw --csv > gpurun_out/prof_c4_raw.csv 2>/dev/null; ls -la gpurun_out/prof_c4*
for c in 2 3 5; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/bench_c$c.json; done
