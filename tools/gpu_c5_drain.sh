# C5 windowed accumulation (MS_T2_DRAIN): batch parity tests, per-contraction time of the
# variants, whole-solve A/B against one accumulator over all of K (dr0), and the accuracy table
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x -p no:cacheprovider > gpurun_out/pytest_batch_drain.log 2>&1; echo rc=$? >> gpurun_out/pytest_batch_drain.log
for i in 1 2; do timeout 300 python tools/tune_tc.py "lib_dr*.so"; done > gpurun_out/tune_drain.log 2>&1
for i in 1 2; do for v in dr2 dr3 dr4 dr0; do
  MS_LIB_PATH=$PWD/paper_2605_23727_b200/_variants/lib_$v.so timeout 600 python tools/bench_c5.py --steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,3), 'M/s', round(d['ms_per_solve'],1), 'ms', d['contraction']['ms'], d['accepted_per_traj_mean'], d['rejected_per_traj_mean'])" >> gpurun_out/c5_drain_ab.log
done; done
for v in dr2 dr3 dr4; do echo "== $v" >> gpurun_out/c5_drain_acc.log; MS_LIB_PATH=$PWD/paper_2605_23727_b200/_variants/lib_$v.so timeout 600 python tools/c5_accuracy.py >> gpurun_out/c5_drain_acc.log 2>&1; done
