export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_configs_full.py tests/test_gpu_batch.py tests/test_gpu_snapshots.py -q -x --timeout 1000 -p no:cacheprovider > gpurun_out/pytest_pow.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_pow.log
for c in c1 c2 c3; do timeout 300 python tools/prof_small.py $c; done > gpurun_out/small.log 2>&1
timeout 600 python tools/bench_c5.py --steps 2 > gpurun_out/c5.log 2>&1
echo done >> gpurun_out/small.log
