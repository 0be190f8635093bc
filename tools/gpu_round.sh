export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python tools/profile_c4.py --kdtype f32 --iters 20 --attempts 1 > gpurun_out/sw.log 2>&1
timeout 300 python tools/profile_c4.py --kdtype f16 --iters 20 --attempts 1 >> gpurun_out/sw.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
