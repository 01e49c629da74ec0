mkdir -p gpurun_out
python -c "import oracle; oracle.build()" >/dev/null 2>&1
for c in 2 3; do for f in 0 1; do TF_FINE=$f timeout 300 python bench.py --config $c --steps 3 --warmup 3 --only --no-e2e --no-cpu 2>/dev/null | tail -1 | cut -c1-160; done; done
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
