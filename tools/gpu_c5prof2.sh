# C5 after the finalize changes: batch suite, launch list (warm caches, host loop), ncu --set full of kb_finalize, bench line
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_batch_sharded_gloo.py -q -x -p no:cacheprovider > gpurun_out/pytest_c5.log 2>&1; echo rc=$? >> gpurun_out/pytest_c5.log
timeout 600 python tools/bench_c5.py > gpurun_out/bench_c5.log 2>&1
MS_LOOP=host timeout 300 python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_host.log 2>&1 && \
MS_LOOP=host timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 40 -c 80 --csv \
  --log-file gpurun_out/c5_launches.csv python tools/bench_c5.py --tf 0.05 --steps 1 > gpurun_out/c5_ncu.log 2>&1
MS_LOOP=host timeout 600 ncu --set full --import-source on --clock-control none -k regex:kb_finalize -s 3 -c 1 -f -o gpurun_out/c5_fin2 \
  python tools/bench_c5.py --tf 0.05 --steps 1 >> gpurun_out/c5_ncu.log 2>&1
echo done
