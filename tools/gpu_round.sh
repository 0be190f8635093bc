export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rhs.py -q -x -k "tile" --timeout 1000 -p no:cacheprovider > gpurun_out/pytest_tile.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_tile.log
for ks in f16 bf16; do timeout 300 python tools/prof_small16.py $ks; done > gpurun_out/c2sweep16.log 2>&1
echo "f16 tile $(MS_SWEEP=tile timeout 300 python tools/profile_c4.py --kdtype f16 --iters 20 --attempts 1 2>&1 | head -1)" >> gpurun_out/c2sweep16.log
