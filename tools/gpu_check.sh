# GPU check after a kernel change: parity suite, then whole C4 solves (f32; f16 register vs TMA sweep, alternating)
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
for i in 1 2; do
  for sw in ldg tma16; do
    MS_SWEEP=$sw timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-accuracy --kdtype f16 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sw f16', d['value'], d['e2e']['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['clocks'].get('power_w'))" >> gpurun_out/ab_f16.log
  done
done
