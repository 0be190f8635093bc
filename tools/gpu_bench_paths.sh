# bench.py paths: sharded loop (N=1 rank), torchrun launch, reference arm at the driver's K/W, f16 line
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
( time timeout 900 python bench.py --shard --steps 2 --warmup 3 --no-cpu-baseline ) > gpurun_out/bench_shard.log 2>&1
( time timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline ) > gpurun_out/bench_torchrun.log 2>&1
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/bench_ref20.log 2>&1
( time timeout 900 python bench.py --kdtype f16 --steps 3 --warmup 3 ) > gpurun_out/bench_f16.log 2>&1
