# C5 contraction: ncu source-level warp-stall sampling (where the issuer, the producer and the drain warps wait)
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
MS_LOOP=host timeout 300 python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_host.log 2>&1 || exit 1
MS_LOOP=host timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tc_gemm2 -s 6 -c 1 -f -o /tmp/c5_tc2 \
  python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_src_ncu.log 2>&1
ncu -i /tmp/c5_tc2.ncu-rep --page source --csv --print-source sass > gpurun_out/c5_tc2_source_sass.csv 2>/dev/null
ncu -i /tmp/c5_tc2.ncu-rep --page details > gpurun_out/c5_tc2_details.txt 2>/dev/null
echo done
