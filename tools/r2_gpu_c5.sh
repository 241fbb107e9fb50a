#!/bin/bash
mkdir -p gpurun_out
for v in main s3n2 s1n4; do
  if [ $v = main ]; then unset SS_LIB_PATH; else export SS_LIB_PATH=$PWD/build_var/lib_$v.so; fi
  echo "$v" >> gpurun_out/c5_bench.log
  timeout 600 python bench.py --cfg 5 --no-cpu-baseline --no-e2e --steps 3 --warmup 2 >> gpurun_out/c5_bench.log 2>&1
done
