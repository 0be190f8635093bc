# the checked build (tools/build_checked.py: -DMS_CHECKS=1) over the small sanitizer cases and the GPU parity tests
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
export MS_LIB_PATH=$PWD/paper_2605_23727_b200/_variants/lib_checked.so
timeout 900 python tools/sanitize_cases.py all > gpurun_out/checked_cases.log 2>&1; echo rc=$? >> gpurun_out/checked_cases.log
timeout 2400 python -m pytest tests/test_gpu_rhs.py tests/test_gpu_solver.py tests/test_gpu_batch.py tests/test_gpu_variants.py \
  tests/test_gpu_edge.py tests/test_gpu_sharded_lockstep.py tests/test_gpu_sharded.py tests/test_gpu_dense.py tests/test_gpu_snapshots.py \
  tests/test_gpu_configs_full.py tests/test_gpu_c4_full.py tests/test_gpu_harness.py tests/test_gpu_tc16.py tests/test_gpu_golden_solves.py tests/test_gpu_acceptance.py -q -p no:cacheprovider > gpurun_out/checked_pytest.log 2>&1; echo rc=$? >> gpurun_out/checked_pytest.log
grep -c "MS_CHECK failed" gpurun_out/checked_pytest.log gpurun_out/checked_cases.log
