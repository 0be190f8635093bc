# round 2, fourth session: ncu evidence of the current tc16 sweep (launch list + --set full of one host-loop attempt)
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
bash tools/gpu_ncu_c4.sh f16
MS_LOOP=host timeout 600 python tools/profile_c4.py --kdtype f16 --iters 1 --attempts 2 > gpurun_out/s4_plain.log 2>&1 || exit 1
MS_LOOP=host timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s4_c4_f16_launches.csv \
  python tools/profile_c4.py --kdtype f16 --iters 1 --attempts 2 > gpurun_out/s4_ncu_list.log 2>&1
echo done
