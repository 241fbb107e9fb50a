#!/bin/bash
# m = 1 composites from the scalar suffix product (k_wsuffix1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_transposed.py -x -q -k "m1 or pseudo or config3 or golden or wide or fark or medium" > gpurun_out/w1_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/w1_pytest.log
timeout 600 python bench.py --cfg 3 --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/w1_bench3.log 2>&1
FUZZ_NMAX=1500 timeout 300 python tools/fuzz_parity.py 31 12 > gpurun_out/w1_fuzz.log 2>&1
echo done
