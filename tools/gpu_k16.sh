# K sweep tuning on C4: burst over every variant (bitwise check), then sustained
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
MS_SWEEP=tma16 timeout 1500 python tools/tune_rhs.py > gpurun_out/tune_k16.txt 2>&1
SW_KS=f16 timeout 900 python tools/sustained_sweep.py ldg:base tma16:base tma16:k16_c8r2_64k tma16:k16_c8r4_64k tma16:k16_c16r2_64k tma16:k16_c16r2_64k_u2 tma16:k16_c16r2_64k_nofadd2 tma16:k16_c12r2_48k > gpurun_out/sus_k16.txt 2>&1
SW_KS=f32 timeout 900 python tools/sustained_sweep.py tma:base tma:u1 tma:u2 tma:u8 tma:nofadd2 tma:base > gpurun_out/sus_f32.txt 2>&1
