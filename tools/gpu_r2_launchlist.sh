# round 2, last session: ncu launch list of the bench command itself (f32 headline, host-driven
# attempt loop so the launches are visible to ncu), after the same command exited 0 without ncu
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-accuracy --no-also"
MS_LOOP=host timeout 900 $CMD > gpurun_out/ll_plain.log 2>&1 || { echo plain_failed; exit 1; }
MS_LOOP=host timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
  --log-file gpurun_out/r2_c4_bench_launches.csv $CMD > gpurun_out/ll_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r2_c4_bench_launches.csv > gpurun_out/r2_c4_bench_launches_summary.txt 2>&1
cat gpurun_out/r2_c4_bench_launches_summary.txt
