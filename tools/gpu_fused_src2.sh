export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for spec in "c1 k_eval_fused" "c1 k_finalize" "c2 k_finalize"; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none --cache-control none -k regex:$2 -s 12 -c 1 -f -o /tmp/src_$1_$2 python tools/prof_small.py $1 > gpurun_out/src_ncu_$1_$2.log 2>&1
  ncu -i /tmp/src_$1_$2.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$1_$2_sass.csv 2>/dev/null
  ncu -i /tmp/src_$1_$2.ncu-rep --page details 2>/dev/null | grep -E "Duration|Grid Size|Block Size|Registers Per" > gpurun_out/src_$1_$2_details.txt
done
echo done
