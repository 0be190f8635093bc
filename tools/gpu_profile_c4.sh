#!/bin/bash
# ncu evidence for the C4 bench line (run under gpurun, one GPU): a full capture
# of one K sweep and the launch list of a whole solve (host loop, so every
# launch is visible), each after the same command has exited 0 without ncu.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python tools/profile_c4.py --iters 4 --attempts 1 > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_rhs_tma -s 1 -c 1 -f -o gpurun_out/tma_f32 \
  python tools/profile_c4.py --iters 4 --attempts 1 > gpurun_out/ncu_full.log 2>&1
MS_LOOP=host python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-accuracy > gpurun_out/bench_host.log 2>&1 || exit 1
MS_LOOP=host ncu --metrics gpu__time_duration.sum --clock-control none -s 9000 -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-accuracy \
  > gpurun_out/ncu_launch.log 2>&1
echo done
