mkdir -p gpurun_out
python -c "import oracle; oracle.build()" >/dev/null 2>&1
for v in 32 default 1024 4096; do
  if [ $v = default ]; then L=""; else L=build/lib_poll$v.so; fi
  for c in 3 2 1 4; do
    r=$(TILEFACT_LIB=$L timeout 600 python bench.py --config $c --steps 5 --warmup 3 --only --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
    echo "poll=$v config=$c ms=$r"
  done
done
