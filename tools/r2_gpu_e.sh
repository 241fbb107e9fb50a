#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fark or group or golden" > gpurun_out/e_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e_pytest.log
for s in 1 2 4 8; do
SS_FARK_SPL=$s timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-reduced > gpurun_out/e_bench4_spl$s.log 2>&1
done
SS_FARK_SPL=4 timeout 600 python bench.py --cfg 2 --no-cpu-baseline --no-e2e > gpurun_out/e_bench2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:k_ --csv --log-file gpurun_out/e_launches_cfg4.csv \
  python bench.py --profile > gpurun_out/e_ncu_list.log 2>&1
echo done
