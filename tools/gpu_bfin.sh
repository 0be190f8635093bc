# C5 finalize reading the last prep's partial x_tilde sum (MS_BFIN_P): A/B and the batch tests
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for i in 1 2; do
  for f in on off; do
    MS_BFIN_P=$f timeout 600 python tools/bench_c5.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['value']), round(d['ms_per_solve'],2))" >> gpurun_out/bfin.log
  done
done
timeout 1200 python -m pytest tests/test_gpu_batch.py tests/test_batch_sharded_gloo.py -q -x -p no:cacheprovider > gpurun_out/pytest_batch.log 2>&1; echo rc=$? >> gpurun_out/pytest_batch.log
