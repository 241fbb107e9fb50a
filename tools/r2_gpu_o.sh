#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for v in main serial; do
  if [ $v = main ]; then unset SS_LIB_PATH; else export SS_LIB_PATH=$PWD/build_var/lib_$v.so; fi
  for nm in "4000 10" "20000 50"; do
    set -- $nm
    echo "$v $1" >> gpurun_out/o_red.log
    timeout 300 python tools/red_probe.py --n $1 --m $2 --p $2 >> gpurun_out/o_red.log 2>&1
  done
done
done
unset SS_LIB_PATH
