# 16-bit K TMA sweep geometry on C4 (burst, bitwise check against base)
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
MS_SWEEP=tma16 timeout 1500 python tools/tune_rhs.py > gpurun_out/tune_k16.txt 2>&1
