mkdir -p gpurun_out
for v in b6 b4 nobulk b6; do
  cp build/variants/$v.so paper_0709_1272_b200/libtilefact.so
  echo "== $v $(timeout 600 python bench.py --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["pct_of_fp64_peak"], d["ms_per_step"])')"
done
