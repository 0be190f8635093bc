#!/bin/bash
# ncu --set full of the K-sweep launches of one host-driven C4 attempt (f32 K:
# k_rhs_tma<.., NEXT=0/1>; f16 K: k_rhs_fast), after the same command exited 0
# without ncu. Exports the raw CSV and the details page into gpurun_out/ (the
# report itself stays in /tmp: gpurun copies back at most 64 MiB).
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
ks=${1:-f32}
MS_LOOP=host python tools/profile_c4.py --kdtype $ks --iters 1 --attempts 1 > gpurun_out/prof_plain_$ks.log 2>&1 || exit 1
MS_LOOP=host ncu --set full --import-source on --clock-control none -k regex:"k_rhs_(tma|fast|tc16)" -c 8 -f \
  -o /tmp/c4_sweeps_$ks python tools/profile_c4.py --kdtype $ks --iters 1 --attempts 1 > gpurun_out/ncu_full_$ks.log 2>&1
ncu -i /tmp/c4_sweeps_$ks.ncu-rep --page raw --csv > gpurun_out/ncu_c4_${ks}_raw.csv 2>/dev/null
ncu -i /tmp/c4_sweeps_$ks.ncu-rep --page details > gpurun_out/ncu_c4_${ks}_details.txt 2>/dev/null
echo ncu_done_$ks
