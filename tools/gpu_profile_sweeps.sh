#!/bin/bash
# ncu --set full of one C4 K sweep per kernel/format (f32 TMA sweep, f16 register
# sweep, f16 TMA sweep), each after the same command has exited 0 without ncu.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python tools/profile_c4.py --iters 4 --attempts 1 > gpurun_out/prof_plain.log 2>&1 || exit 1
python tools/profile_c4.py --iters 4 --attempts 1 --kdtype f16 >> gpurun_out/prof_plain.log 2>&1 || exit 1
MS_SWEEP=tma16 python tools/profile_c4.py --iters 4 --attempts 1 --kdtype f16 >> gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_rhs_tma -s 1 -c 1 -f -o gpurun_out/tma_f32 \
  python tools/profile_c4.py --iters 4 --attempts 1 > gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_rhs_fast -s 1 -c 1 -f -o gpurun_out/ldg_f16 \
  python tools/profile_c4.py --iters 4 --attempts 1 --kdtype f16 >> gpurun_out/ncu_full.log 2>&1
MS_SWEEP=tma16 ncu --set full --import-source on --clock-control none -k regex:k_rhs_tma -s 1 -c 1 -f -o gpurun_out/tma_f16 \
  python tools/profile_c4.py --iters 4 --attempts 1 --kdtype f16 >> gpurun_out/ncu_full.log 2>&1
echo done
