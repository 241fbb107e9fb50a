#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_farkd --launch-skip 10 --launch-count 1 \
  -o /tmp/dm3_c5 -f python bench.py --cfg 5 --profile > gpurun_out/dm3_ncu5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_farkd --launch-skip 10 --launch-count 1 \
  -o /tmp/dm3_c2 -f python bench.py --cfg 2 --profile > gpurun_out/dm3_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_farkd --launch-skip 40 --launch-count 1 \
  -o /tmp/dm3_c4 -f python bench.py --profile > gpurun_out/dm3_ncu4.log 2>&1
python tools/ncu_summary.py - /tmp/dm3_c4.ncu-rep /tmp/dm3_c2.ncu-rep /tmp/dm3_c5.ncu-rep > gpurun_out/dm3_summary.txt 2>&1
for c in 2 4 5; do
ncu -i /tmp/dm3_c$c.ncu-rep --page source --csv --print-source sass > gpurun_out/dm3_sass$c.csv 2>/dev/null
done
echo done
