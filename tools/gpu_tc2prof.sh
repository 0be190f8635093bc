# ncu --set full (with source) of one C5 stage contraction, after a clean run
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
MS_LOOP=host timeout 300 python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_host.log 2>&1 && \
MS_LOOP=host ncu --set full --import-source on --clock-control none -k regex:k_tc_gemm2 -s 12 -c 1 -f -o gpurun_out/tc2 \
  python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/tc2_ncu.log 2>&1
echo done
