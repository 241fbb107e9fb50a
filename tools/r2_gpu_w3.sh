#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "wide or golden or medium or config5" > gpurun_out/w3_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/w3_pytest.log
timeout 900 python -m pytest tests/test_gpu_transposed.py tests/test_gpu_irka.py -x -q >> gpurun_out/w3_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/w3_pytest.log
timeout 600 python bench.py --cfg 5 --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > gpurun_out/w3_bench5.log 2>&1
timeout 300 python tools/lq_probe.py --n 10000 --m 20 --s 2000 >> gpurun_out/w3_lq.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum \
  --clock-control none -k regex:k_wsuffix --launch-count 5 --csv --log-file gpurun_out/w3_wsuf.csv \
  python bench.py --cfg 5 --profile > /dev/null 2>&1
echo done
