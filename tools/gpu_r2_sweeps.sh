# round 2: sustained C4 sweep A/B of the packed-product kernels vs the round-1 build, then sharded/golden tests
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded_lockstep.py tests/test_gpu_golden_solves.py -k "c2 or row_shards" -q -x -p no:cacheprovider > gpurun_out/pytest_lockstep.log 2>&1; echo rc=$? >> gpurun_out/pytest_lockstep.log
SW_KS=f16 timeout 1200 python tools/sustained_sweep.py ldg ldg:r1 ldg:fr4 ldg:fr12 ldg:fr16 ldg:fr8_t256 tma16 tma16:r1 tma16:pk_c16r2 tma16:pk_c8r2 tma16:pk_c4r8 tma16:pk_c8r8 tma16:pk_c8r4_32k_s6 > gpurun_out/sweeps_f16.log 2>&1
SW_KS=f32 timeout 600 python tools/sustained_sweep.py tma tma:r1 tma:pk_sss_c4r4 tma:pk_sss_c4r2 > gpurun_out/sweeps_f32.log 2>&1
