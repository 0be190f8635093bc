set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo rc=$? >> gpurun_out/bench_full.log
timeout 600 python bench.py --steps 2 --warmup 1 --kdtype f16 --no-cpu-baseline > gpurun_out/bench_f16.log 2>&1; echo rc=$? >> gpurun_out/bench_f16.log
timeout 600 python tools/bench_c5.py > gpurun_out/c5_tc.log 2>&1; echo rc=$? >> gpurun_out/c5_tc.log
CMD="python tools/profile_c4.py --iters 4 --attempts 1"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rhs_tma -s 2 -c 1 -o gpurun_out/prof_rhs_tma $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$? >> gpurun_out/prof_plain.log
CMD2="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-accuracy"
export MS_LOOP=host
timeout 300 $CMD2 > gpurun_out/plain_hostloop.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 9000 -c 3000 --csv --log-file gpurun_out/launches_hostloop.csv $CMD2 > gpurun_out/ncu_launch.log 2>&1
echo ncu2_rc=$? >> gpurun_out/plain_hostloop.log
