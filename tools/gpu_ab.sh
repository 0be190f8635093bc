mkdir -p gpurun_out
for i in 1 2; do
for v in new old; do
  if [ $v = old ]; then export MS_LIB_PATH=$PWD/paper_2605_23727_b200/_variants/lib_tf_sss_c16r1.so; else unset MS_LIB_PATH; fi
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-accuracy 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['e2e']['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['clocks']['power_w'])" >> gpurun_out/ab.log
done; done
