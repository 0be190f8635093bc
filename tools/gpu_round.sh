export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for c in c1 c2 c3; do timeout 300 python tools/prof_small.py $c; done > gpurun_out/small.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_configs_full.py -q -x --timeout 1000 -p no:cacheprovider > gpurun_out/pytest_s.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_s.log
echo done >> gpurun_out/small.log
