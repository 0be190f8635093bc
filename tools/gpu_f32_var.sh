export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for i in 1 2; do SW_KS=f32 timeout 900 python tools/sustained_sweep.py tma:cur tma:r1 tma:f32_nopk tma:f32_pk_u2 tma:f32_pk_u8 tma:f32_pk_c16r1 tma:f32_pk_c8r4 tma:f32_pk_s3; done > gpurun_out/sweeps_f32_var.log 2>&1
