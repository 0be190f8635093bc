# prep loops rolled (MS_PREP_ROLL): C1-C3 per-attempt A/B, C4 f32 solve A/B, tests with the default build
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out; rm -f gpurun_out/roll_ab.log gpurun_out/roll_c4.log
V=$PWD/paper_2605_23727_b200/_variants
timeout 1500 python -m pytest tests/test_gpu_solver.py tests/test_gpu_edge.py tests/test_gpu_rhs.py tests/test_gpu_configs_full.py tests/test_gpu_snapshots.py -m gpu -q -x -p no:cacheprovider > gpurun_out/roll_tests.log 2>&1; echo rc=$? >> gpurun_out/roll_tests.log
for i in 1 2 3; do for v in roll0 roll1; do
  MS_LIB_PATH=$V/lib_$v.so timeout 600 python tools/ab_small.py $v >> gpurun_out/roll_ab.log 2>&1
done; done
for i in 1 2; do for v in roll0 roll1; do
  MS_LIB_PATH=$V/lib_$v.so timeout 600 python bench.py --no-cpu-baseline --no-also --no-accuracy --steps 3 --warmup 3 2>/dev/null | grep '^{"metric' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); r = d['roofline']
    print('$v', 'f32', round(d['value'], 2), round(d['e2e']['value'], 2), round(r['solve_effective_GBps'], 1), round(r['launch_ms'], 4), d['clocks']['sm_mhz'])
" >> gpurun_out/roll_c4.log
done; done
echo done
