# fourth session: per-k-block full barriers (MS_GV_KBFULL) and accumulator batch variants
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
V=$PWD/paper_2605_23727_b200/_variants
MS_LIB_PATH=$V/lib_gv_kbfull.so timeout 900 python -m pytest tests/test_gpu_tc16.py -m gpu -q -x -p no:cacheprovider > gpurun_out/tc16_kbfull_tests.log 2>&1; echo rc=$? >> gpurun_out/tc16_kbfull_tests.log
rm -f gpurun_out/tc16_var2.log
for i in 1 2; do for v in ${VARS:-gv_new gv_kbfull gv_kbfull_z gv_g8b2}; do
  MS_SWEEP=tc16 MS_LIB_PATH=$V/lib_$v.so timeout 300 python tools/profile_c4.py --kdtype f16 --iters 20 --attempts 1 2>&1 | grep "rhs" | sed "s/^/$v /" >> gpurun_out/tc16_var2.log
done; done
echo done
