#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/d_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/d_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/d_bench4.log 2>&1
timeout 600 python bench.py --cfg 2 --no-cpu-baseline --no-e2e > gpurun_out/d_bench2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:k_ --csv --log-file gpurun_out/d_launches_cfg4.csv \
  python bench.py --profile > gpurun_out/d_ncu_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fark --launch-skip 1 --launch-count 1 \
  -o gpurun_out/d_fark_cfg4 -f python bench.py --profile > gpurun_out/d_ncu_fark.log 2>&1
echo done
