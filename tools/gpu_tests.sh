mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
export TF_DIST_TIMEOUT_S=30
timeout 2400 python -m pytest tests -q -m gpu -x --durations=8 2>&1 | tail -25 | tee gpurun_out/pytest_gpu_full.log
