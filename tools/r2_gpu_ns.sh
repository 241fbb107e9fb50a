#!/bin/bash
# wide-window composites on two streams (two halves of the batch)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "wide or config5 or golden or batch or isolation" > gpurun_out/ns_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ns_pytest.log
timeout 600 python bench.py --cfg 5 --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > gpurun_out/ns_bench5.log 2>&1
echo done
