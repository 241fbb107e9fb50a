#!/bin/bash
# two-level sweep with the batch's halves on two streams (comparison build ns2tl)
mkdir -p gpurun_out
for v in main ns2tl; do
  if [ $v = main ]; then unset SS_LIB_PATH; else export SS_LIB_PATH=$PWD/build_var/lib_$v.so; fi
  for c in 4 2; do
    echo "$v cfg$c" >> gpurun_out/ns2_bench.log
    timeout 600 python bench.py --cfg $c --no-cpu-baseline --no-e2e --steps 3 --warmup 2 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['frac'],d.get('reduced') and d['reduced']['value'])" >> gpurun_out/ns2_bench.log 2>&1
  done
done
export SS_LIB_PATH=$PWD/build_var/lib_ns2tl.so
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "two_level or golden or batch or deferred or medium" > gpurun_out/ns2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ns2_pytest.log
