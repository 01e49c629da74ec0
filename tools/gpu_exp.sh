python -c "import oracle; oracle.build()"
timeout 900 python tools/emu_bench.py --config 4 --grids 1x1,1x2,2x2,2x4 2>&1 | tail -2
timeout 900 python tools/emu_bench.py --config 5 --grids 1x1,1x2,1x4 2>&1 | tail -2
