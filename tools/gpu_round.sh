export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python tools/bench_c5.py --steps 2 > gpurun_out/c5_tc.log 2>&1
timeout 300 python tools/bench_c5.py --tf 2.0 --steps 1 > gpurun_out/c5_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python tools/bench_c5.py --tf 2.0 --steps 1 > gpurun_out/ncu_launch_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kb_finalize" -s 5 -c 1 -o gpurun_out/prof_c5_fin2 -f python tools/bench_c5.py --tf 2.0 --steps 1 > gpurun_out/ncu_c5_fin.log 2>&1
echo done >> gpurun_out/ncu_c5_fin.log
