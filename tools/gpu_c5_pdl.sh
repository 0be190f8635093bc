# C5: early dependent-launch release in the contraction (MS_TC_PDL=late restores the release at exit)
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -q -x -p no:cacheprovider > gpurun_out/pytest_batch3.log 2>&1; echo rc=$? >> gpurun_out/pytest_batch3.log
for i in 1 2; do for e in early late; do
  MS_TC_PDL=$e timeout 600 python tools/bench_c5.py --steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$e', round(d['value']/1e6,3), 'M/s', round(d['ms_per_solve'],1), 'ms', d['contraction']['ms'])" >> gpurun_out/c5_pdl_ab.log
done; done
