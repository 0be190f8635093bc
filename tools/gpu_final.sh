# end-of-round check of the committed build: full GPU suite, smoke, bench (C4 f32 + f16), reference arm, configs
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 2700 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 900 python bench.py --kdtype f16 --no-cpu-baseline > gpurun_out/bench_f16.log 2>&1; echo rc=$? >> gpurun_out/bench_f16.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_ref.log
timeout 600 python tools/ab_small.py final > gpurun_out/configs_final.log 2>&1
echo done
