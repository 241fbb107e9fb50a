#!/bin/bash
mkdir -p gpurun_out
for spl in 4 8 16 37; do for c in 5 3; do
  echo "spl $spl cfg$c" >> gpurun_out/x_bench.log
  SS_SPL=$spl timeout 600 python bench.py --cfg $c --no-cpu-baseline --no-e2e --steps 3 --warmup 2 >> gpurun_out/x_bench.log 2>&1
done; done
