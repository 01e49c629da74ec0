mkdir -p gpurun_out
python -c "import oracle; oracle.build()" >/dev/null 2>&1
for v in 0 4 8 16; do
  for c in 3 2 1; do
    r=$(TF_RESERVE=$v timeout 600 python bench.py --config $c --steps 5 --warmup 3 --only --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
    echo "reserve=$v config=$c ms=$r"
  done
done
