set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python tools/tune_tc.py > gpurun_out/tune_tc.log 2>&1; echo rc=$? >> gpurun_out/tune_tc.log
