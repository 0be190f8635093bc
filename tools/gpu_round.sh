export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_edge.py -q -x -k cooperative --timeout 120 -p no:cacheprovider > gpurun_out/pytest_coop.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_coop.log
for c in c1 c2 c3; do timeout 120 python tools/prof_small.py $c | grep graph; done > gpurun_out/small.log 2>&1
echo done >> gpurun_out/small.log
