export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rhs.py -q -x --timeout 1000 -p no:cacheprovider > gpurun_out/pytest_rhs.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_rhs.log
timeout 900 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
