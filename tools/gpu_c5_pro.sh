# C5 contraction: relaxed prologue pair barrier (MS_T2_PRO_RELAXED) -- tests, golden gate, speed A/B
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out; rm -f gpurun_out/c5_pro_*.log
V=$PWD/paper_2605_23727_b200/_variants
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x -p no:cacheprovider > gpurun_out/c5_pro_batch.log 2>&1; echo rc=$? >> gpurun_out/c5_pro_batch.log
timeout 900 python -m pytest tests/test_gpu_golden_solves.py -k c5 -q -x -s -p no:cacheprovider > gpurun_out/c5_pro_golden.log 2>&1; echo rc=$? >> gpurun_out/c5_pro_golden.log
for i in 1 2 3; do for v in t2_pro0 t2_pro1; do
  MS_LIB_PATH=$V/lib_$v.so timeout 600 python tools/bench_c5.py --steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,3), 'M/s', round(d['ms_per_solve'],1), 'ms', round(d['contraction']['ms']*1e3,2), 'us')" >> gpurun_out/c5_pro_ab.log
done; done
echo done
