export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_harness.py -q -x --timeout 800 -p no:cacheprovider > gpurun_out/pytest_var.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_var.log
timeout 900 python tools/bench_variants.py --c4-tf 5.0 > gpurun_out/bench_variants.log 2>&1
echo done >> gpurun_out/bench_variants.log
