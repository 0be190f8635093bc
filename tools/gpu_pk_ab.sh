# packed FMUL2.FTZ sweeps: parity suite, then whole C4 solves A/B (MS_SWEEP_PK=off = scalar products)
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_golden_solves.py -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
for i in 1 2; do
  for pk in on off; do
    for ks in f32 f16; do
      MS_SWEEP_PK=$pk timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-accuracy --kdtype $ks 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$pk $ks', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['achieved']), d['roofline']['launch_ms'], d['clocks']['sm_mhz'], d['clocks'].get('power_w'))" >> gpurun_out/ab_pk.log
    done
  done
done
