export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for i in 1 2; do for v in tcv_base tcv_rec64 tcv_stcg tcv_fin tcv_noepi r1; do timeout 300 python tools/tune_tc.py "lib_$v.so"; done; done > gpurun_out/tune_tc_r2b.log 2>&1
