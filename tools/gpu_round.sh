set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 120 python tools/tc_smoke.py > gpurun_out/tc_smoke.log 2>&1; echo rc=$? >> gpurun_out/tc_smoke.log
timeout 900 python -m pytest tests/test_gpu_batch.py -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_batch.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_batch.log
timeout 600 python tools/bench_c5.py > gpurun_out/c5_tc.log 2>&1; echo rc=$? >> gpurun_out/c5_tc.log
CMD="python tools/bench_c5.py --tf 0.5 --steps 1"
export MS_LOOP=host
timeout 300 $CMD > gpurun_out/c5_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 5 -c 1 -o gpurun_out/prof_tc_gemm2 $CMD > gpurun_out/ncu_tc.log 2>&1
echo ncu_rc=$? >> gpurun_out/c5_plain.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 600 --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/ncu_launch_c5.log 2>&1
echo ncu2_rc=$? >> gpurun_out/c5_plain.log
