# C5 accumulation windows (MS_TC_WINDOW k-blocks; 32 = one accumulator over all of K):
# batch tests, full-size golden gate, whole-solve speed and accuracy per window
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x -p no:cacheprovider > gpurun_out/pytest_batch_win.log 2>&1; echo rc=$? >> gpurun_out/pytest_batch_win.log
timeout 900 python -m pytest tests/test_gpu_golden_solves.py -k c5 -q -x -s -p no:cacheprovider > gpurun_out/pytest_c5_win.log 2>&1; echo rc=$? >> gpurun_out/pytest_c5_win.log
for i in 1 2; do for wv in 2 3 4 32; do
  MS_TC_WINDOW=$wv timeout 600 python tools/bench_c5.py --steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('window $wv', round(d['value']/1e6,3), 'M/s', round(d['ms_per_solve'],1), 'ms', d['contraction']['ms'])" >> gpurun_out/c5_window_ab.log
done; done
for wv in 2 3 32; do echo "== window $wv" >> gpurun_out/c5_window_acc.log; MS_TC_WINDOW=$wv timeout 600 python tools/c5_accuracy.py >> gpurun_out/c5_window_acc.log 2>&1; done
