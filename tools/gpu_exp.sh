python -c "import oracle; oracle.build()"
export TF_DIST_TIMEOUT_S=30
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
