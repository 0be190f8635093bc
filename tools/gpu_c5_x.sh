export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for i in 1 2; do for v in tcv_noepi tcx_halfb tcx_nob tcx_1mma tcx_0mma; do timeout 300 python tools/tune_tc.py "lib_$v.so"; done; done > gpurun_out/tune_tc_x.log 2>&1
