# C5 finalize geometry: 128-thread trajectory blocks (64 registers, unrolled element loop) vs 256 x 32 registers
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
V=paper_2605_23727_b200/_variants
for i in 1 2; do
  for v in base fin_t128_u4 fin_t128_u8 fin_t128; do
    if [ $v = base ]; then L=""; else L="MS_LIB_PATH=$V/lib_$v.so"; fi
    env $L timeout 600 python tools/bench_c5.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_solve'],2))" >> gpurun_out/ab_bfin2.log
  done
done
MS_LIB_PATH=$V/lib_fin_t128_u4.so timeout 900 python -m pytest tests/test_gpu_batch.py -q -x -p no:cacheprovider > gpurun_out/pytest_bfin2.log 2>&1; echo rc=$? >> gpurun_out/pytest_bfin2.log
echo done
