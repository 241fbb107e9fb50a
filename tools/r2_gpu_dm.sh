#!/bin/bash
# k_farkd (DMMA far pass, m = 20): parity + config-4 timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "two_level or fark or golden or medium or config1 or block_groups or paired or deferred or config4 or streamed" > gpurun_out/dm_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/dm_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > gpurun_out/dm_bench4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum \
  --clock-control none -k regex:k_fark --launch-skip 30 --launch-count 3 --csv --log-file gpurun_out/dm_fark.csv \
  python bench.py --profile > /dev/null 2>&1
echo done
