# round-2 check after the tc16 sweep: full GPU suite, smoke, ncu capture of the f16 C4 sweeps
# (tc16), bench lines (C4 f32, C4 f16), C5
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
bash tools/gpu_ncu_c4.sh f16 > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 900 python bench.py --kdtype f16 --no-cpu-baseline > gpurun_out/bench_f16.log 2>&1; echo rc=$? >> gpurun_out/bench_f16.log
timeout 600 python tools/bench_c5.py --steps 2 > gpurun_out/bench_c5.log 2>&1
echo done
