# C5 contraction: 128-bit record loads + global stores in the epilogue vs round 1
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -q -x -p no:cacheprovider > gpurun_out/pytest_batch2.log 2>&1; echo rc=$? >> gpurun_out/pytest_batch2.log
for i in 1 2; do timeout 300 python tools/tune_tc.py "lib_cur.so"; timeout 300 python tools/tune_tc.py "lib_r1.so"; done > gpurun_out/tune_tc_r2.log 2>&1
for i in 1 2; do timeout 600 python tools/bench_c5.py --steps 2 | tail -1 >> gpurun_out/c5_bench_r2.log 2>&1; done
