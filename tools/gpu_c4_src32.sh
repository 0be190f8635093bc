# C4 f32 row-copy sweep: ncu source-level warp sampling of k_rhs_tma<float, float, 1, 1>
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
MS_LOOP=host timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_rhs_tma<float, float" -s 1 -c 1 -f \
  -o /tmp/c4src_f32 python tools/profile_c4.py --kdtype f32 --iters 1 --attempts 1 > gpurun_out/c4src_ncu_f32.log 2>&1
ncu -i /tmp/c4src_f32.ncu-rep --page source --csv --print-source sass > gpurun_out/c4src_f32_sass.csv 2>/dev/null
ncu -i /tmp/c4src_f32.ncu-rep --page details > gpurun_out/c4src_f32_details.txt 2>/dev/null
echo done
