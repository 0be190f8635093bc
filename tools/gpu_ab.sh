#!/bin/bash
# Whole C4 solves (bench.py --steps 5) alternating between build variants on one
# box: bash tools/gpu_ab.sh <variant> [<variant> ...]  ("default" = the in-tree
# library; others = paper_2605_23727_b200/_variants/lib_<name>.so). Appends
# "name value e2e in-solve-GB/s sm_mhz power_w" lines to gpurun_out/ab.log.
mkdir -p gpurun_out
for i in 1 2; do
  for v in "$@"; do
    if [ "$v" = default ]; then unset MS_LIB_PATH; else export MS_LIB_PATH=$PWD/paper_2605_23727_b200/_variants/lib_$v.so; fi
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-accuracy --kdtype ${KDTYPE:-f32} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v ${KDTYPE:-f32}', d['value'], d['e2e']['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['clocks']['power_w'])" >> gpurun_out/ab.log
  done
done
