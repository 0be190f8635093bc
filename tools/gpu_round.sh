export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
export MS_LOOP=host
timeout 300 python tools/bench_c5.py --tf 0.5 --steps 1 > gpurun_out/c5s.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tc_gemm2" -s 10 -c 1 -o gpurun_out/prof_tc2_final -f python tools/bench_c5.py --tf 0.5 --steps 1 > gpurun_out/ncu_tc2.log 2>&1
timeout 300 python tools/prof_variants.py c4 > gpurun_out/pv.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rhs_multi" -s 6 -c 1 -o gpurun_out/prof_multi_final -f python tools/prof_variants.py c4 > gpurun_out/ncu_multi.log 2>&1
timeout 300 python tools/prof_small.py c1 > gpurun_out/ps.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_eval_fused" -s 20 -c 1 -o gpurun_out/prof_fused_final -f python tools/prof_small.py c1 > gpurun_out/ncu_fused.log 2>&1
echo done
