#!/bin/bash
mkdir -p gpurun_out
for v in main occ12 occ16; do
  if [ $v = main ]; then unset SS_LIB_PATH; else export SS_LIB_PATH=$PWD/build_var/lib_$v.so; fi
  for c in 2 4; do
    echo "$v cfg$c" >> gpurun_out/s_bench.log
    timeout 600 python bench.py --cfg $c --no-cpu-baseline --no-e2e --no-reduced >> gpurun_out/s_bench.log 2>&1
  done
done
