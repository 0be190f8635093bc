# launch lists (ncu durations, cold-cache, serialised) of a few host-loop attempts of C1/C2/C3 + graph-loop per-attempt time
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for c in c1 c2 c3; do
  timeout 300 python tools/prof_small.py $c > gpurun_out/small_${c}_plain.log 2>&1 || exit 1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/small_${c}_launches.csv python tools/prof_small.py $c > gpurun_out/small_${c}_ncu.log 2>&1
done
echo done
