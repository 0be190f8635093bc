export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for g in 8 6 4 2 1; do echo "gridn=$g"; MS_T2_GRIDN=$g timeout 300 python tools/tune_tc.py "lib_tcv_noepi.so"; MS_T2_GRIDN=$g timeout 300 python tools/tune_tc.py "lib_cur.so"; done > gpurun_out/tune_tc_grid.log 2>&1
