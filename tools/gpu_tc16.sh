# f16-K tensor-core sweep (MS_SWEEP=tc16): parity tests (incl. the whole C4 f16 solve vs the
# oracle fixture), per-launch sweep time (burst), then whole C4 f16 solves against the
# default register sweep, alternating on one box
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc16.py -q -x -p no:cacheprovider -s > gpurun_out/pytest_tc16.log 2>&1; echo rc=$? >> gpurun_out/pytest_tc16.log
grep -q "rc=0" gpurun_out/pytest_tc16.log || exit 1
for sw in tc16 ldg; do MS_SWEEP=$sw timeout 300 python tools/profile_c4.py --kdtype f16 --iters 20 --attempts 1 2>&1 | grep "rhs" | sed "s/^/$sw /" >> gpurun_out/sw_tc16.log; done
for i in 1 2; do for sw in tc16 default; do
  if [ $sw = default ]; then unset MS_SWEEP; else export MS_SWEEP=$sw; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-accuracy --kdtype f16 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sw f16', d['value'], d['e2e']['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['clocks'].get('power_w'), d.get('accepted_steps_per_solve'), d.get('rejected_per_solve'))" >> gpurun_out/ab_tc16.log
done; done
unset MS_SWEEP
