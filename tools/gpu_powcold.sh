# controller code size: the general pow path and libm pow out of line (MS_POW_COLD) -- C1-C3 per-attempt time A/B + solver tests
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out; rm -f gpurun_out/powcold_ab.log
V=$PWD/paper_2605_23727_b200/_variants
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_edge.py -m gpu -q -x -p no:cacheprovider > gpurun_out/powcold_tests.log 2>&1; echo rc=$? >> gpurun_out/powcold_tests.log
for i in 1 2 3; do for v in pow_cold0 pow_cold1; do
  MS_LIB_PATH=$V/lib_$v.so timeout 600 python tools/ab_small.py $v >> gpurun_out/powcold_ab.log 2>&1
done; done
echo done
