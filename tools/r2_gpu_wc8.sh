#!/bin/bash
mkdir -p gpurun_out
for v in main wc8; do
  if [ $v = main ]; then unset SS_LIB_PATH; else export SS_LIB_PATH=$PWD/build_var/lib_$v.so; fi
  echo "$v" >> gpurun_out/wc8_bench.log
  timeout 600 python bench.py --cfg 3 --no-cpu-baseline --no-e2e --steps 5 --warmup 3 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['frac'])" >> gpurun_out/wc8_bench.log 2>&1
done
