mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -40 | tee gpurun_out/pytest_gpu1.log
