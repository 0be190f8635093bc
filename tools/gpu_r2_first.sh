export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_ref.log
bash tools/gpu_ncu_c4.sh f32
timeout 900 python -m pytest tests/test_bench_contract.py tests/test_gpu_c4_full.py tests/test_abi.py -q -x > gpurun_out/pytest_part.log 2>&1; echo rc=$? >> gpurun_out/pytest_part.log
