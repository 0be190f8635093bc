# C5 contraction: relaxed drain arrive (MS_T2_DRAIN_RELAXED) -- tests, golden gate, speed A/B per window
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out; rm -f gpurun_out/c5_rel_*.log
V=$PWD/paper_2605_23727_b200/_variants
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x -p no:cacheprovider > gpurun_out/c5_rel_batch.log 2>&1; echo rc=$? >> gpurun_out/c5_rel_batch.log
timeout 900 python -m pytest tests/test_gpu_golden_solves.py -k c5 -q -x -s -p no:cacheprovider > gpurun_out/c5_rel_golden.log 2>&1; echo rc=$? >> gpurun_out/c5_rel_golden.log
for i in 1 2; do for v in t2_rel0 t2_rel1; do for wv in 2 3 4; do
  MS_LIB_PATH=$V/lib_$v.so MS_TC_WINDOW=$wv timeout 600 python tools/bench_c5.py --steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v window $wv', round(d['value']/1e6,3), 'M/s', round(d['ms_per_solve'],1), 'ms', round(d['contraction']['ms']*1e3,2), 'us')" >> gpurun_out/c5_rel_ab.log
done; done; done
echo done
