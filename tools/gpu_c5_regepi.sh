# C5: coupling epilogue from the drain warps' registers (MS_T2_REGEPI) vs totals back to TMEM + 8-warp epilogue
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x -p no:cacheprovider > gpurun_out/pytest_batch_rege.log 2>&1; echo rc=$? >> gpurun_out/pytest_batch_rege.log
for i in 1 2; do timeout 300 python tools/tune_tc.py "lib_rege*.so"; done > gpurun_out/tune_rege.log 2>&1
for i in 1 2; do for v in rege1 rege0; do
  MS_LIB_PATH=$PWD/paper_2605_23727_b200/_variants/lib_$v.so timeout 600 python tools/bench_c5.py --steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,3), 'M/s', round(d['ms_per_solve'],1), 'ms', d['contraction']['ms'])" >> gpurun_out/c5_rege_ab.log
done; done
timeout 900 python -m pytest tests/test_gpu_golden_solves.py -k c5 -q -x -s -p no:cacheprovider > gpurun_out/pytest_c5_rege.log 2>&1; echo rc=$? >> gpurun_out/pytest_c5_rege.log
