# two resident TMA-sweep CTAs per SM (smaller rings): C2 attempt time and C4 burst per variant
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for i in 1 2; do
  for v in base tma_m2_32k_s3 tma_m2_48k_s2 tma_m2_24k_s4; do
    export MS_LIB_PATH=$PWD/paper_2605_23727_b200/_variants/lib_$v.so
    echo "== $v" >> gpurun_out/m2.log
    timeout 300 python tools/c2_attempt_time.py 2>&1 | grep f32 >> gpurun_out/m2.log
  done
done
unset MS_LIB_PATH
timeout 1200 python tools/tune_rhs.py > gpurun_out/m2_tune.txt 2>&1
