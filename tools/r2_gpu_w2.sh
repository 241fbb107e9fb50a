#!/bin/bash
# k_wsuffix profile at config 5 (launch list + one full capture)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:k_ --csv --log-file gpurun_out/w2_launches_cfg5.csv \
  python bench.py --cfg 5 --profile > gpurun_out/w2_ncu_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wsuffix --launch-skip 5 --launch-count 1 \
  -o /tmp/w2_wsuf -f python bench.py --cfg 5 --profile > gpurun_out/w2_ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/w2_launches_cfg5.csv /tmp/w2_wsuf.ncu-rep > gpurun_out/w2_summary.txt 2>&1
ncu -i /tmp/w2_wsuf.ncu-rep --page source --csv > gpurun_out/w2_wsuf_source.csv 2>/dev/null
echo done
