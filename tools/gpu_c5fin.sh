# C5 finalize: ncu --set full of kb_finalize (host loop so ncu sees it), after a clean run
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
MS_LOOP=host timeout 300 python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5fin_host.log 2>&1 && \
MS_LOOP=host timeout 600 ncu --set full --import-source on --clock-control none -k regex:kb_finalize -s 3 -c 1 -f -o gpurun_out/c5_fin \
  python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5fin_ncu.log 2>&1
echo done
