# round 2, fourth session: tc16 issuer / prologue / combine variants
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
V=$PWD/paper_2605_23727_b200/_variants
timeout 900 python -m pytest tests/test_gpu_tc16.py -m gpu -q -x -p no:cacheprovider > gpurun_out/tc16_tests.log 2>&1; echo rc=$? >> gpurun_out/tc16_tests.log
rm -f gpurun_out/tc16_var.log
for i in 1 2; do for v in ${VARS:-gv_old gv_u gv_uc gv_new gv_new_fine gv_new_fine_i1 gv_new_kb2 gv_new_zatom}; do
  MS_SWEEP=tc16 MS_LIB_PATH=$V/lib_$v.so timeout 300 python tools/profile_c4.py --kdtype f16 --iters 20 --attempts 1 2>&1 | grep "rhs" | sed "s/^/$v /" >> gpurun_out/tc16_var.log
done; done
rm -f gpurun_out/tc16_solve_ab.log
for i in 1 2; do for v in ${SOLVE_VARS:-gv_old gv_new}; do
  MS_LIB_PATH=$V/lib_$v.so timeout 600 python bench.py --kdtype f16 --no-cpu-baseline --no-also --steps 3 --warmup 3 2>&1 | grep '^{"metric' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); r = d['roofline']
    print('$v', 'f16', round(d['value'], 2), round(d['e2e']['value'], 2), round(r['solve_effective_GBps'], 1), round(r['launch_ms'], 4), d['clocks']['sm_mhz'], d['clocks'].get('power_w'), d['accepted_steps_per_solve'], d['rejected_per_solve'])
" >> gpurun_out/tc16_solve_ab.log
done; done
echo done
