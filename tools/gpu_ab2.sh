mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
for v in k16s4 k32s3 k16s5; do
  cp build/variants/$v.so paper_0709_1272_b200/libtilefact.so
  P=$(timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1)
  echo "== $v $(timeout 600 python bench.py --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["pct_of_fp64_peak"], d["ms_per_step"])') | $P"
done
