# one-block finalize threshold (MS_FIN_SMALL_MAX 2048 default vs 4096 / 8192) now that the controller runs on a shared Ctl copy
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
V=paper_2605_23727_b200/_variants
for i in 1 2; do
  timeout 600 python tools/ab_small.py base >> gpurun_out/ab_finsmall.log 2>&1
  MS_LIB_PATH=$V/lib_fin_small4k.so timeout 600 python tools/ab_small.py small4k >> gpurun_out/ab_finsmall.log 2>&1
  MS_LIB_PATH=$V/lib_fin_small8k.so timeout 600 python tools/ab_small.py small8k >> gpurun_out/ab_finsmall.log 2>&1
done
echo done
