#!/bin/bash
mkdir -p gpurun_out
for g in 4 8; do for c in 4 2; do
  echo "group $g cfg$c" >> gpurun_out/w_bench.log
  SS_GROUP=$g timeout 600 python bench.py --cfg $c --no-cpu-baseline --no-e2e >> gpurun_out/w_bench.log 2>&1
done; done
SS_GROUP=8 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or config1 or two_level or group or medium" > gpurun_out/w_pytest.log 2>&1; echo rc=$? >> gpurun_out/w_pytest.log
