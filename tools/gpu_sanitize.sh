# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over tools/sanitize_cases.py
export PYTHONUNBUFFERED=1; mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize_cases.py c2_f32 > gpurun_out/sanitize/plain.log 2>&1; echo rc=$? >> gpurun_out/sanitize/plain.log
for tool in memcheck synccheck racecheck initcheck; do
  for c in c2_f32 c2_f16 c2_policies c1_fused c3_fused faithful dense_snapshots variants batch_tc batch_cuda_cores dp54 sharded_one_rank; do
    extra=""
    [ $tool = memcheck ] && extra="--leak-check full"
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 300 $CS --tool $tool $extra --target-processes all --print-limit 50 \
      python tools/sanitize_cases.py $c > gpurun_out/sanitize/${tool}_$c.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' gpurun_out/sanitize/${tool}_$c.log | tr '\n' ' ')" >> gpurun_out/sanitize/summary.txt
  done
done
