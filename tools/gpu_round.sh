export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_configs_full.py tests/test_gpu_c4_full.py -q -s --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_repro.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_repro.log
timeout 600 python -m pytest tests/test_gpu_c4_full.py -q -s --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_repro2.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_repro2.log
timeout 120 python tools/profile_c4.py --n 4096 --iters 2 --attempts 1 > gpurun_out/san_plain.log 2>&1 && \
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/profile_c4.py --n 4096 --iters 2 --attempts 1 > gpurun_out/racecheck.log 2>&1
echo san_rc=$? >> gpurun_out/san_plain.log
