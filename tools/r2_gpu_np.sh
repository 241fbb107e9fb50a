#!/bin/bash
# near updates (128 rows) on the pass kernels instead of the K-streamed kernel
mkdir -p gpurun_out
for v in main np128; do
  if [ $v = main ]; then unset SS_LIB_PATH; else export SS_LIB_PATH=$PWD/build_var/lib_$v.so; fi
  for c in 4 2; do
    echo "$v cfg$c" >> gpurun_out/np_bench.log
    timeout 600 python bench.py --cfg $c --no-cpu-baseline --no-e2e --steps 3 --warmup 2 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['frac'],d.get('reduced') and d['reduced']['value'])" >> gpurun_out/np_bench.log 2>&1
  done
done
export SS_LIB_PATH=$PWD/build_var/lib_np128.so
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "two_level or golden or medium or deferred or groups" > gpurun_out/np_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/np_pytest.log
