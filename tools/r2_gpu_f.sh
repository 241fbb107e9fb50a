#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/f_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/f_bench4.log 2>&1
echo done
