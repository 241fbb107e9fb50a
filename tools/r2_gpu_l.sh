#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "reduc or hess or config1 or corpus or criterion or golden" > gpurun_out/l_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/l_pytest.log
for nm in "1500 10" "2000 1" "4000 10" "10000 20" "20000 50"; do
  set -- $nm
  timeout 300 python tools/red_probe.py --n $1 --m $2 --p $2 >> gpurun_out/l_red.log 2>&1
done
