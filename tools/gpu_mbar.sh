# mbarrier try loop rolled (MS_MBAR_ROLL): C1-C3 per-attempt A/B, C4 f32 solve A/B, per-launch sweep
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out; rm -f gpurun_out/mbar_ab.log gpurun_out/mbar_c4.log gpurun_out/mbar_launch.log
V=$PWD/paper_2605_23727_b200/_variants
for i in 1 2 3; do for v in mbar0 mbar1; do
  MS_LIB_PATH=$V/lib_$v.so timeout 600 python tools/ab_small.py $v >> gpurun_out/mbar_ab.log 2>&1
  MS_LIB_PATH=$V/lib_$v.so timeout 300 python tools/profile_c4.py --iters 20 --attempts 1 2>&1 | grep "rhs" | sed "s/^/$v /" >> gpurun_out/mbar_launch.log
done; done
for i in 1 2; do for v in mbar0 mbar1; do
  MS_LIB_PATH=$V/lib_$v.so timeout 600 python bench.py --no-cpu-baseline --no-also --no-accuracy --steps 3 --warmup 3 2>/dev/null | grep '^{"metric' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); r = d['roofline']
    print('$v', 'f32', round(d['value'], 2), round(d['e2e']['value'], 2), round(r['solve_effective_GBps'], 1), round(r['launch_ms'], 4), d['clocks']['sm_mhz'])
" >> gpurun_out/mbar_c4.log
done; done
echo done
