# C5 per-kernel durations (warm caches, serialised) of host-loop attempts, after a clean run
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
MS_LOOP=host timeout 300 python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_host.log 2>&1 && \
MS_LOOP=host ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 40 -c 80 --csv \
  --log-file gpurun_out/c5_launches.csv python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_ncu.log 2>&1
MS_LOOP=host ncu --set full --import-source on --clock-control none -k regex:kb_prep_tc -s 3 -c 1 -f -o gpurun_out/c5_prep \
  python tools/bench_c5.py --tf 0.05 --steps 1 >> gpurun_out/c5_ncu.log 2>&1
echo done
