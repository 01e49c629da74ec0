mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
for a in "gemm 512 64 1 8" "gemm 1024 64 1 4" "syrk 512 64 1 8" "trsm 512 64 1 4" "potrf 512 64 1 2" "ssrfb 256 32 1 4" "ssrfb 512 64 1 2" "ssssm 256 32 1 4" "tsqrt 256 32 1 2"; do timeout 60 ./build/kbench $a; done 2>&1 | tee gpurun_out/kb7.jsonl
for v in mb sync; do
  cp build/variants/$v.so paper_0709_1272_b200/libtilefact.so
  P=$(timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1)
  echo "== $v $(timeout 600 python bench.py --steps 3 --warmup 2 --only --no-e2e --no-cpu 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["pct_of_fp64_peak"], d["ms_per_step"])') | $P"
done
