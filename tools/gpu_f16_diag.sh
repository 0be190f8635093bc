# f16 K sweep diagnosis: sustained rates (new vs round-1 build) and one ncu --set full capture per sweep kernel
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rhs.py -q -x -k "packed or bitwise" -p no:cacheprovider > gpurun_out/pytest_rhs.log 2>&1; echo rc=$? >> gpurun_out/pytest_rhs.log
SW_KS=f16 timeout 900 python tools/sustained_sweep.py ldg ldg:r1 tma16 > gpurun_out/sweeps_f16b.log 2>&1
for sw in ldg tma16; do
  MS_SWEEP=$sw timeout 300 python tools/profile_c4.py --kdtype f16 --iters 2 --attempts 0 > gpurun_out/prof16_$sw.log 2>&1
  MS_SWEEP=$sw timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_rhs_(tma|fast)" -s 1 -c 1 -f \
    -o gpurun_out/k16_$sw python tools/profile_c4.py --kdtype f16 --iters 2 --attempts 0 > gpurun_out/ncu16_$sw.log 2>&1
done
