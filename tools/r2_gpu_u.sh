#!/bin/bash
mkdir -p gpurun_out
for v in main s3n4 s5n3 s6n2; do
  if [ $v = main ]; then unset SS_LIB_PATH; else export SS_LIB_PATH=$PWD/build_var/lib_$v.so; fi
  echo "$v" >> gpurun_out/u_bench.log
  timeout 600 python bench.py --cfg 4 --no-cpu-baseline --no-e2e --no-reduced >> gpurun_out/u_bench.log 2>&1
done
