#!/bin/bash
# k_fark<2,4,4> (config 4) source-level capture
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fark --launch-skip 40 --launch-count 1 \
  -o /tmp/fk -f python bench.py --profile > gpurun_out/fk_ncu.log 2>&1
python tools/ncu_summary.py - /tmp/fk.ncu-rep > gpurun_out/fk_summary.txt 2>&1
ncu -i /tmp/fk.ncu-rep --page source --csv --print-source sass > gpurun_out/fk_sass.csv 2>/dev/null
ncu -i /tmp/fk.ncu-rep --page details --csv > gpurun_out/fk_details.csv 2>/dev/null
echo done
