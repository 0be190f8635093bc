# f16 tensor-core sweep variants: per-launch time of the C4 sweep (tools/profile_c4.py, 20 evaluations)
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
V=$PWD/paper_2605_23727_b200/_variants
for i in 1 2; do for v in ${VARS:-gv_cur gv_fine_i1 gv_fine_i2 gv_fine_i4}; do
  MS_SWEEP=tc16 MS_LIB_PATH=$V/lib_$v.so timeout 300 python tools/profile_c4.py --kdtype f16 --iters 20 --attempts 1 2>&1 | grep "rhs" | sed "s/^/$v /" >> gpurun_out/tc16_var.log
done; done
