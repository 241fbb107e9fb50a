#!/bin/bash
# full-set capture of four consecutive k_fark launches of config 4 (one group:
# three near updates + the far pass), summarised
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fark --launch-skip 36 --launch-count 4 \
  -o /tmp/ff -f python bench.py --profile > gpurun_out/ff_ncu.log 2>&1
python tools/ncu_summary.py - /tmp/ff.ncu-rep > gpurun_out/ff_summary.txt 2>&1
echo done
