# C5 A/B: in-tree library vs build variants (tools/build_variants.py), alternating; then the batch GPU tests
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for i in 1 2; do
  for v in default "$@"; do
    if [ "$v" = default ]; then unset MS_LIB_PATH; else export MS_LIB_PATH=$PWD/paper_2605_23727_b200/_variants/lib_$v.so; fi
    timeout 600 python tools/bench_c5.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['contraction']; print('$v', round(d['value']), round(d['ms_per_solve'],2), round(c['ms']*1e3,2), round(c['prep_ms']*1e3,2))" >> gpurun_out/c5ab.log
  done
done
unset MS_LIB_PATH
timeout 1200 python -m pytest tests/test_gpu_batch.py tests/test_batch_sharded_gloo.py -q -x -p no:cacheprovider > gpurun_out/pytest_batch.log 2>&1; echo rc=$? >> gpurun_out/pytest_batch.log
