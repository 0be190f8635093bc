# controller on a shared-memory copy of Ctl (MS_CTL_SMEM): parity suites, then A/B
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_solver.py tests/test_gpu_batch.py tests/test_gpu_edge.py tests/test_gpu_sharded.py tests/test_gpu_dense.py tests/test_gpu_snapshots.py -q -x -p no:cacheprovider > gpurun_out/pytest_ctl.log 2>&1; echo rc=$? >> gpurun_out/pytest_ctl.log
for i in 1 2; do
  for v in on off; do
    MS_CTL_SMEM=$v timeout 600 python tools/ab_small.py $v >> gpurun_out/ab_ctl_small.log 2>&1
    MS_CTL_SMEM=$v timeout 600 python tools/bench_c5.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_solve'],2))" >> gpurun_out/ab_ctl_c5.log
  done
done
echo done
