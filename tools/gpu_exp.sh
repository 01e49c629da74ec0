python -c "import oracle; oracle.build()"
for k in getrf tstrf gessm ssssm; do ./build/kbench_lu $k 256 32 1 4; done
for k in gessm ssssm; do ./build/kbench_lu $k 512 64 1 4; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k lu 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k config3 2>&1 | tail -1
for c in 3; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>&1 | tail -1 | cut -c100-190; done
