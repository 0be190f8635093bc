# round-2 ncu evidence: C4 K-sweep captures (f32 TMA + folded prep, f16 register sweep), C5 finalize and contraction
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
bash tools/gpu_ncu_c4.sh f32
bash tools/gpu_ncu_c4.sh f16
MS_LOOP=host timeout 300 python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_host2.log 2>&1 && \
MS_LOOP=host ncu --set full --import-source on --clock-control none --cache-control none -k regex:"kb_finalize|k_tc_gemm2" -s 6 -c 2 -f \
  -o /tmp/c5_fin_gemm python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_ncu2.log 2>&1
ncu -i /tmp/c5_fin_gemm.ncu-rep --page raw --csv > gpurun_out/c5_fin_gemm_raw.csv 2>/dev/null
ncu -i /tmp/c5_fin_gemm.ncu-rep --page details > gpurun_out/c5_fin_gemm_details.txt 2>/dev/null
ncu -i /tmp/c5_fin_gemm.ncu-rep --page source --csv -k regex:kb_finalize > gpurun_out/c5_fin_source.csv 2>/dev/null
du -sh gpurun_out
echo done
