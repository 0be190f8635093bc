# C2 attempt time per K-sweep kernel / geometry variant, alternating
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for i in 1 2; do
  for v in default ldg tf_sss_c16r1 tf_sss_c16r1_32k_s6 tf_sss_32k_s6 tf_sss_16k_s8; do
    unset MS_LIB_PATH MS_SWEEP
    if [ "$v" = ldg ]; then export MS_SWEEP=ldg; elif [ "$v" != default ]; then export MS_LIB_PATH=$PWD/paper_2605_23727_b200/_variants/lib_$v.so; fi
    echo "== $v" >> gpurun_out/c2var.log
    timeout 300 python tools/c2_attempt_time.py 2>&1 | grep f32 >> gpurun_out/c2var.log
  done
done
