# whole C4 solves, this build vs the round-1 build, alternating; C5 finalize source-level capture
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 1500 python tools/ab_solve.py f16 cur r1 > gpurun_out/ab_r1_f16.log 2>&1
timeout 1500 python tools/ab_solve.py f32 cur r1 > gpurun_out/ab_r1_f32.log 2>&1
MS_LOOP=host ncu --set full --import-source on --clock-control none --cache-control none -k regex:kb_finalize -s 3 -c 1 -f \
  -o /tmp/c5_fin python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_fin_ncu.log 2>&1
ncu -i /tmp/c5_fin.ncu-rep --page details > gpurun_out/c5_fin_details.txt 2>/dev/null
ncu -i /tmp/c5_fin.ncu-rep --page source --csv > gpurun_out/c5_fin_source.csv 2>/dev/null
