# the whole -m gpu suite (the round-end driver's check), with timing per test
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 ${PYTEST_K:+-k "$PYTEST_K"} -s > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu_full.log
