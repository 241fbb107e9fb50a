#!/bin/bash
mkdir -p gpurun_out
for v in main u2 u8 ro ro8; do
  if [ $v = main ]; then unset SS_LIB_PATH; else export SS_LIB_PATH=$PWD/build_var/lib_$v.so; fi
  echo "$v" >> gpurun_out/uv_bench.log
  timeout 600 python bench.py --cfg 4 --no-cpu-baseline --no-e2e --no-reduced >> gpurun_out/uv_bench.log 2>&1
done
