# k_finalize (single solve, C1 and C2): ncu source-level sampling in a host-loop run
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for c in c1 c2; do
  timeout 600 ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_finalize -s 8 -c 1 -f -o /tmp/fin_$c python tools/prof_small.py $c > gpurun_out/fin_ncu_$c.log 2>&1
  ncu -i /tmp/fin_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/fin_${c}_sass.csv 2>/dev/null
  ncu -i /tmp/fin_$c.ncu-rep --page details > gpurun_out/fin_${c}_details.txt 2>/dev/null
done
echo done
