export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rhs.py -q -x -k "fused" --timeout 1000 -p no:cacheprovider > gpurun_out/pytest_fused.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_fused.log
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
for c in c1 c2 c3; do timeout 300 python tools/prof_small.py $c; MS_FUSE=off timeout 300 python tools/prof_small.py $c; done > gpurun_out/small.log 2>&1
echo done >> gpurun_out/small.log
