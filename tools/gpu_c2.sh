# C2 (Kuramoto N = 4096, K in L2) per-kernel durations with warm caches
# (ncu --cache-control none) of host-loop attempts, after a clean run
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
MS_LOOP=host python tools/profile_c4.py --n 4096 --iters 4 --attempts 40 > /dev/null 2>&1 && \
MS_LOOP=host ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 60 -c 120 --csv \
  --log-file gpurun_out/c2_launches.csv python tools/profile_c4.py --n 4096 --iters 4 --attempts 40 > gpurun_out/c2_ncu.log 2>&1
MS_LOOP=host ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 60 -c 120 --csv \
  --log-file gpurun_out/c2_launches_f16.csv python tools/profile_c4.py --n 4096 --iters 4 --attempts 40 --kdtype f16 >> gpurun_out/c2_ncu.log 2>&1
echo done
