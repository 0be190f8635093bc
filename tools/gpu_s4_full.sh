# fourth session: tc16 grid experiment, then the full GPU suite + smoke + bench lines of the current build
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out; rm -f gpurun_out/tc16_grid.log
for i in 1 2; do for gsz in 148 128 144; do
  MS_GV_GRID=$gsz MS_SWEEP=tc16 timeout 300 python tools/profile_c4.py --kdtype f16 --iters 20 --attempts 1 2>&1 | grep "rhs" | sed "s/^/grid $gsz /" >> gpurun_out/tc16_grid.log
done; done
bash tools/gpu_final.sh
