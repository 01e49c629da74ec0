# Panel-level Cholesky DAG: bitwise / trace tests, then config 4 with the tile-level (TF_FINE=0)
# and the panel-level (default) graph back to back.
mkdir -p gpurun_out
python -c "import oracle; oracle.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_slab_dag.py tests/test_gpu_trace.py -q -m gpu -x 2>&1 | tail -5
for f in 0 1; do
  TF_FINE=$f timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --only --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/c4_fine$f.json
  echo "fine=$f: $(cut -c1-260 gpurun_out/c4_fine$f.json)"
done
