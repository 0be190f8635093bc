export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rhs.py tests/test_gpu_c4_full.py tests/test_gpu_configs_full.py tests/test_gpu_sharded.py -q -x --timeout 1000 -p no:cacheprovider > gpurun_out/pytest_sw.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_sw.log
timeout 900 python bench.py --kdtype f16 --no-cpu-baseline > gpurun_out/bench_f16.log 2>&1; echo rc=$? >> gpurun_out/bench_f16.log
for ks in f16 bf16; do timeout 300 python tools/prof_small16.py $ks; done > gpurun_out/c2sweep16.log 2>&1
