set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
MS_SWEEP=tma timeout 1200 python tools/tune_rhs.py > gpurun_out/tune_tma2.log 2>&1; echo rc=$? >> gpurun_out/tune_tma2.log
timeout 900 python -m pytest tests/test_gpu_c4_full.py tests/test_gpu_batch.py tests/test_gpu_rhs.py -q -s --timeout 600 -p no:cacheprovider > gpurun_out/pytest_b.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_b.log
