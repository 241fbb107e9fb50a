#!/bin/bash
# k_farkd for m = 10 / 20 / 40 / 50 / 60: full GPU suite + configs 2, 4, 5
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/dm2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/dm2_pytest.log
for c in 4 2 5; do
  timeout 600 python bench.py --cfg $c --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > gpurun_out/dm2_bench$c.log 2>&1
done
echo done
