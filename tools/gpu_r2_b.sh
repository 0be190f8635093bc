# round 2: reference-order kernel (k_rhs_seq) tests, c2 golden gates, f16 register-sweep variants
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rhs.py tests/test_gpu_solver.py tests/test_gpu_configs_full.py -q -x -p no:cacheprovider > gpurun_out/pytest_b1.log 2>&1; echo rc=$? >> gpurun_out/pytest_b1.log
timeout 900 python -m pytest tests/test_gpu_golden_solves.py -k "c2" -q -p no:cacheprovider -s > gpurun_out/pytest_b2.log 2>&1; echo rc=$? >> gpurun_out/pytest_b2.log
SW_KS=f16 timeout 900 python tools/sustained_sweep.py ldg ldg:pf_t384 ldg:pf_t256 ldg:pf_r4 ldg:pf_r6_t384 ldg:t384 ldg:r12_t384 > gpurun_out/sweeps_f16c.log 2>&1
