# Round evidence: every bench line on one box (C4 f32 / f16, reference arm, C5, C1-C3, concurrent variants)
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out/ev
timeout 900 python bench.py > gpurun_out/ev/bench_c4.log 2>&1
timeout 900 python bench.py --kdtype f16 > gpurun_out/ev/bench_c4_f16.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev/bench_ref.log 2>&1
timeout 900 python tools/bench_c5.py > gpurun_out/ev/c5.log 2>&1
timeout 1800 python tools/bench_configs.py > gpurun_out/ev/configs.log 2>&1
timeout 1200 python tools/bench_variants.py > gpurun_out/ev/variants.log 2>&1
echo done
