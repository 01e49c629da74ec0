# All bench configs (1 GPU) + the default bench line, for BASELINE.md §5 / profiles.
mkdir -p gpurun_out
python -c "import oracle; oracle.build()" >/dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/res_smi.txt
for c in 1 2 3 5 6; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --only --no-cpu 2>gpurun_out/res_c$c.err | tail -1 > gpurun_out/res_c$c.json; echo "c$c rc=$?"; done
timeout 1200 python bench.py > gpurun_out/res_c4.json 2> gpurun_out/res_c4.err; echo "c4 rc=$?"
