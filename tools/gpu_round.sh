set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 120 python tools/tc_smoke.py > gpurun_out/tc_smoke.log 2>&1; echo rc=$? >> gpurun_out/tc_smoke.log
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_sharded.py -q --timeout 300 -x -p no:cacheprovider > gpurun_out/pytest_batch.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_batch.log
