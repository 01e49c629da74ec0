# Round-end check (one gpurun call): the whole GPU suite, smoke, every bench config, the
# default bench line (config 4 with e2e and the CPU baseline), the reference arm, then the
# config-4 ncu launch list and one --set full capture of tf_persistent.
mkdir -p gpurun_out
python -c "import oracle; oracle.build()" >/dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/final_smi.txt
timeout 2400 python -m pytest tests -q -m gpu -rA > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/final_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in 1 2 3 5 6; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --only --no-cpu 2>gpurun_out/final_c$c.err | tail -1 > gpurun_out/final_c$c.json; echo "c$c rc=$? $(cut -c100-230 gpurun_out/final_c$c.json)"; done
timeout 1200 python bench.py > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err; echo "c4 rc=$? $(cut -c100-230 gpurun_out/final_c4.json)"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$? $(cut -c1-200 gpurun_out/final_ref.json)"
TAG=${TAG:-r02d}
CMD="python bench.py --steps 1 --warmup 1 --only --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$TAG.csv $CMD > gpurun_out/ncu_launch_c4.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tf_persistent -s 1 -c 1 -o gpurun_out/prof_c4_$TAG $CMD > gpurun_out/ncu_full_c4.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/prof_c4_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_c4_${TAG}_raw.csv 2>/dev/null
