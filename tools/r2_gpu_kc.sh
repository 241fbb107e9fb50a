#!/bin/bash
# k_fark m = 20 chunk width / unit shape variants (config 4, config 2)
mkdir -p gpurun_out
for v in main kc16s4n4 kc16s4n7 kc16s6n5; do
  if [ $v = main ]; then unset SS_LIB_PATH; else export SS_LIB_PATH=$PWD/build_var/lib_$v.so; fi
  for c in 4 2; do
    echo "$v cfg$c" >> gpurun_out/kc_bench.log
    timeout 600 python bench.py --cfg $c --no-cpu-baseline --no-e2e --steps 3 --warmup 2 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['frac'])" >> gpurun_out/kc_bench.log 2>&1
  done
done
echo done
