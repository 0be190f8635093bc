# fourth session: unit-end ticket as one acq_rel atomic after a barrier (MS_GV_ATOMREL)
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
V=$PWD/paper_2605_23727_b200/_variants
timeout 1500 python -m pytest tests/test_gpu_tc16.py tests/test_gpu_sharded_lockstep.py tests/test_gpu_golden_solves.py -m gpu -q -x -p no:cacheprovider -k "tc16 or f16" > gpurun_out/tc16_ar_tests.log 2>&1; echo rc=$? >> gpurun_out/tc16_ar_tests.log
rm -f gpurun_out/tc16_ar.log gpurun_out/tc16_ar_solve.log
for i in 1 2 3; do for v in gv_ar0 gv_ar1 gv_ar1_own1; do
  MS_SWEEP=tc16 MS_LIB_PATH=$V/lib_$v.so timeout 300 python tools/profile_c4.py --kdtype f16 --iters 20 --attempts 1 2>&1 | grep "rhs" | sed "s/^/$v /" >> gpurun_out/tc16_ar.log
done; done
for i in 1 2; do for v in gv_ar0 gv_ar1; do
  MS_LIB_PATH=$V/lib_$v.so timeout 600 python bench.py --kdtype f16 --no-cpu-baseline --no-also --steps 3 --warmup 3 2>/dev/null | grep '^{"metric' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); r = d['roofline']
    print('$v', 'f16', round(d['value'], 2), round(d['e2e']['value'], 2), round(r['solve_effective_GBps'], 1), round(r['launch_ms'], 4), d['clocks']['sm_mhz'], d['clocks'].get('power_w'), d['accepted_steps_per_solve'], d['rejected_per_solve'])
" >> gpurun_out/tc16_ar_solve.log
done; done
echo done
