export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_edge.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_edge.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_edge.log
