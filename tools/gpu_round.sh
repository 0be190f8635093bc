set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --maxfail=40 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-accuracy"
export MS_LOOP=host
timeout 300 $CMD > gpurun_out/plain_hostloop.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 9000 -c 3000 --csv --log-file gpurun_out/launches_hostloop.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo ncu_rc=$? >> gpurun_out/plain_hostloop.log
