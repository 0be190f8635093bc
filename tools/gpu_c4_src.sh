# C4 sweeps: ncu source-level warp sampling (f16 tensor-core sweep, f32 row-copy sweep)
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for ks in f16 f32; do
  MS_LOOP=host timeout 300 python tools/profile_c4.py --kdtype $ks --iters 1 --attempts 1 > gpurun_out/c4src_plain_$ks.log 2>&1 || exit 1
  MS_LOOP=host timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_rhs_(tma|tc16)" -s 3 -c 1 -f \
    -o /tmp/c4src_$ks python tools/profile_c4.py --kdtype $ks --iters 1 --attempts 1 > gpurun_out/c4src_ncu_$ks.log 2>&1
  ncu -i /tmp/c4src_$ks.ncu-rep --page source --csv --print-source sass > gpurun_out/c4src_${ks}_sass.csv 2>/dev/null
done
echo done
