# k_finalize instruction footprint: element loop unroll 4 vs 1 (MS_FIN_UNROLL) -- C1-C3 per-attempt time A/B + tests
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out; rm -f gpurun_out/finu_ab.log
V=$PWD/paper_2605_23727_b200/_variants
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_edge.py tests/test_gpu_configs_full.py -m gpu -q -x -p no:cacheprovider > gpurun_out/finu_tests.log 2>&1; echo rc=$? >> gpurun_out/finu_tests.log
for i in 1 2 3; do for v in fin_u4 fin_u1; do
  MS_LIB_PATH=$V/lib_$v.so timeout 600 python tools/ab_small.py $v >> gpurun_out/finu_ab.log 2>&1
done; done
echo done
