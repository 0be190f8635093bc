export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x --timeout 800 -p no:cacheprovider > gpurun_out/pytest_batch.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_batch.log
timeout 600 python tools/bench_c5.py --steps 2 > gpurun_out/c5.log 2>&1
