#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none --launch-skip 3000 --launch-count 400 --csv --log-file gpurun_out/m_red20k.csv \
  python tools/red_probe.py --n 20000 --m 50 --p 50 --profile > gpurun_out/m_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/m_red20k.csv > gpurun_out/m_sum.txt 2>&1
