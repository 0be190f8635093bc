export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python tools/tune_tc.py "lib_tc2_*.so" > gpurun_out/tune_tc2b.log 2>&1
timeout 900 python tools/tune_tc.py "lib_tc2_*.so" >> gpurun_out/tune_tc2b.log 2>&1
