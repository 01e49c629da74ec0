mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "rc=$?"
tail -5 gpurun_out/bench1.err
cat gpurun_out/bench1.json
