# folded next-stage prep (MS_FUSE_NEXT): C2 attempt time and C4 whole solves, on/off alternating; then the GPU suite
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for i in 1 2; do
  for f in on off; do
    echo "== $f" >> gpurun_out/fuse.log
    MS_FUSE_NEXT=$f timeout 300 python tools/c2_attempt_time.py 2>&1 | grep f32 >> gpurun_out/fuse.log
    MS_FUSE_NEXT=$f timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-accuracy 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4', d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])" >> gpurun_out/fuse.log
  done
done
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
