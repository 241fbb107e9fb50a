#!/bin/bash
# two far-kernel CTAs per SM (k_fark<2,2,NST>, 4 consumer warps each) vs one
mkdir -p gpurun_out
for v in main c2s2n3 c2s2n2; do
  if [ $v = main ]; then unset SS_LIB_PATH; else export SS_LIB_PATH=$PWD/build_var/lib_$v.so; fi
  echo "$v" >> gpurun_out/c2_bench.log
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['frac'])" >> gpurun_out/c2_bench.log 2>&1
done
cuobjdump -res-usage build_var/lib_c2s2n3.so 2>/dev/null | grep -A1 "k_farkILi2ELi2E" | tail -1 >> gpurun_out/c2_bench.log
