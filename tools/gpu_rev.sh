# tc16 unit-order reversal on alternate launches: per-launch sweep time and whole C4 f16 solves
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
V=$PWD/paper_2605_23727_b200/_variants
for i in 1 2; do for v in ${VARS:-gv_rev0 gv_rev1}; do
  MS_SWEEP=tc16 MS_LIB_PATH=$V/lib_$v.so timeout 300 python tools/profile_c4.py --kdtype f16 --iters 20 --attempts 1 2>&1 | grep "rhs" | sed "s/^/$v /" >> gpurun_out/rev.log
done; done
for i in 1 2; do for v in ${VARS:-gv_rev0 gv_rev1}; do
  MS_LIB_PATH=$V/lib_$v.so timeout 600 python bench.py --kdtype f16 --steps 3 --warmup 2 --no-cpu-baseline --no-accuracy --no-also 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', round(d['value'],2), round(d['e2e']['value'],2), d['roofline'].get('solve_effective_GBps'), d['clocks']['sm_mhz'], d.get('accepted_steps_per_solve'), d.get('rejected_per_solve'))
" >> gpurun_out/rev.log
done; done
