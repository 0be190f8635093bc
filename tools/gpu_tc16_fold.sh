# round 2, fourth session: the tensor-core sweep folds the next stage's prep (k_rhs_tc16<NEXT>)
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tc16.py tests/test_gpu_solver.py tests/test_gpu_sharded_lockstep.py tests/test_gpu_golden_solves.py -m gpu -q -x -p no:cacheprovider -k "tc16 or f16 or fold or push" > gpurun_out/tc16_fold_tests.log 2>&1; echo rc=$? >> gpurun_out/tc16_fold_tests.log
rm -f gpurun_out/tc16_fold_ab.log
for i in 1 2; do for f in off on; do
  MS_FUSE_NEXT=$f timeout 600 python bench.py --kdtype f16 --no-cpu-baseline --no-also --steps 3 --warmup 3 2>gpurun_out/tc16_fold_err_$f.log | grep '^{"metric' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); r = d['roofline']
    print('fold=$f', 'f16', round(d['value'], 2), round(d['e2e']['value'], 2), round(r['solve_effective_GBps'], 1), round(r['launch_ms'], 4), d['clocks']['sm_mhz'], d['clocks'].get('power_w'), d['accepted_steps_per_solve'], d['rejected_per_solve'], d['gpu_launches'])
" >> gpurun_out/tc16_fold_ab.log
done; done
echo done
