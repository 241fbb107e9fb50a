#!/bin/bash
mkdir -p gpurun_out
for cfg in "96 6" "64 6" "64 8" "56 8" "48 8" "48 10" "32 12"; do
  set -- $cfg
  echo "nb $1 win $2" >> gpurun_out/k_bench5.log
  SS_WC_NB=$1 SS_WC_WIN=$2 timeout 600 python bench.py --cfg 5 --no-cpu-baseline --no-e2e --steps 3 --warmup 1 >> gpurun_out/k_bench5.log 2>&1
done
