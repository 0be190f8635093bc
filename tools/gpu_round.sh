export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python tools/bench_c5.py --steps 2 --kdtype f16 > gpurun_out/c5_f16.log 2>&1
timeout 600 python tools/bench_c5.py --steps 2 --kdtype bf16 > gpurun_out/c5_bf16.log 2>&1
timeout 600 python tools/bench_c5.py --steps 1 --tc 0 > gpurun_out/c5_cc.log 2>&1
timeout 300 python -m pytest tests/test_cpp_api.py -q -p no:cacheprovider > gpurun_out/pytest_cpp.log 2>&1; echo rc=$? >> gpurun_out/pytest_cpp.log
