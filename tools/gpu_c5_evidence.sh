# C5 evidence for the windowed-accumulation build: warm-cache launch list of host-loop
# attempts, and ncu --set full of one stage contraction (after a clean run)
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
MS_LOOP=host timeout 300 python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_host.log 2>&1 || exit 1
MS_LOOP=host ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 40 -c 80 --csv \
  --log-file gpurun_out/c5_launches.csv python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/c5_launches.csv > gpurun_out/c5_launches_summary.txt 2>&1
MS_LOOP=host ncu --set full --import-source on --clock-control none -k regex:k_tc_gemm2 -s 12 -c 1 -f -o /tmp/tc2w \
  python tools/bench_c5.py --tf 0.05 --steps 1 >> gpurun_out/c5_ncu.log 2>&1
ncu -i /tmp/tc2w.ncu-rep --page details > gpurun_out/tc2w_details.txt 2>/dev/null
ncu -i /tmp/tc2w.ncu-rep --page raw --csv > gpurun_out/tc2w_raw.csv 2>/dev/null
echo done
