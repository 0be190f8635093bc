# QuotMax (finalize without per-element division): tests, C5 whole-solve A/B, launch list; golden C4 gates
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_batch.py tests/test_gpu_golden_solves.py -k "not c5_full" -q -p no:cacheprovider -s > gpurun_out/pytest_c.log 2>&1; echo rc=$? >> gpurun_out/pytest_c.log
for i in 1 2; do for e in on off; do
  MS_BFIN_QUOT=$e timeout 600 python tools/bench_c5.py --steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('quot=$e', round(d['value']/1e6,3), 'M/s', round(d['ms_per_solve'],1), 'ms', d['contraction']['ms'])" >> gpurun_out/c5_quot_ab.log
done; done
MS_LOOP=host timeout 300 python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_host3.log 2>&1 && \
MS_LOOP=host ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 40 -c 80 --csv \
  --log-file gpurun_out/c5_launches3.csv python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_ncu3.log 2>&1
python tools/launch_summary.py gpurun_out/c5_launches3.csv > gpurun_out/c5_launches3_summary.txt 2>&1
