# C5 contraction A/B: epilogue records staged in shared memory (MS_T2_SREC) and the
# relaxed end-of-kernel pair barrier (MS_T2_END_RELAXED) vs the previous kernel
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x -p no:cacheprovider > gpurun_out/pytest_batch_srec.log 2>&1; echo rc=$? >> gpurun_out/pytest_batch_srec.log
for i in 1 2; do timeout 300 python tools/tune_tc.py "lib_tcs_*.so"; done > gpurun_out/tune_tc_srec.log 2>&1
for i in 1 2; do for v in tcs_new tcs_old; do
  MS_LIB_PATH=$PWD/paper_2605_23727_b200/_variants/lib_$v.so timeout 600 python tools/bench_c5.py --steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,3), 'M/s', round(d['ms_per_solve'],1), 'ms', d['contraction']['ms'])" >> gpurun_out/c5_srec_ab.log
done; done
