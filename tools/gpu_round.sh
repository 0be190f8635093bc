export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dense.py tests/test_gpu_snapshots.py tests/test_gpu_solver.py tests/test_gpu_variants.py -q -x --timeout 1000 -p no:cacheprovider > gpurun_out/pytest_dense.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_dense.log
