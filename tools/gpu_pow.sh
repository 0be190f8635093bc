# controller pow started from sqrt/cbrt instead of libm pow (MS_POW_ROOT_START): A/B
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
V=paper_2605_23727_b200/_variants
for i in 1 2; do
  timeout 600 python tools/ab_small.py root >> gpurun_out/ab_pow_small.log 2>&1
  MS_LIB_PATH=$V/lib_pow_libm_api.so timeout 600 python tools/ab_small.py libm >> gpurun_out/ab_pow_small.log 2>&1
  timeout 600 python tools/bench_c5.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('root', round(d['value']), round(d['ms_per_solve'],2))" >> gpurun_out/ab_pow_c5.log
  MS_LIB_PATH=$V/lib_pow_libm_batch.so timeout 600 python tools/bench_c5.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('libm', round(d['value']), round(d['ms_per_solve'],2))" >> gpurun_out/ab_pow_c5.log
done
timeout 1500 python -m pytest tests/test_gpu_solver.py tests/test_gpu_batch.py tests/test_gpu_configs_full.py -q -x -p no:cacheprovider > gpurun_out/pytest_pow.log 2>&1; echo rc=$? >> gpurun_out/pytest_pow.log
echo done
