export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for i in 1 2; do timeout 300 python tools/tune_tc.py "lib_dr*.so"; done > gpurun_out/tune_drain2.log 2>&1
for i in 1 2; do for v in dr2x8 dr3x8 dr2 dr0; do
  MS_LIB_PATH=$PWD/paper_2605_23727_b200/_variants/lib_$v.so timeout 600 python tools/bench_c5.py --steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,3), 'M/s', round(d['ms_per_solve'],1), 'ms', d['contraction']['ms'])" >> gpurun_out/c5_drain_ab2.log
done; done
