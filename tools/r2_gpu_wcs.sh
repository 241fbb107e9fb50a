#!/bin/bash
# config 5 window-composite shape (windows x width) with suffix composites + two streams
mkdir -p gpurun_out
for v in main w10n48 w12n40 w16n32; do
  if [ $v = main ]; then unset SS_LIB_PATH; else export SS_LIB_PATH=$PWD/build_var/lib_$v.so; fi
  echo "$v" >> gpurun_out/wcs_bench.log
  timeout 600 python bench.py --cfg 5 --no-cpu-baseline --no-e2e --steps 3 --warmup 2 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['frac'])" >> gpurun_out/wcs_bench.log 2>&1
done
