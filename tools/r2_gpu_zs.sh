#!/bin/bash
# branch-free W22e selects in k_farkd's state part
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/zs_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/zs_pytest.log
for c in 4 5 2; do timeout 600 python bench.py --cfg $c --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > gpurun_out/zs_bench$c.log 2>&1; done
echo done
