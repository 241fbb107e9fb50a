#!/bin/bash
mkdir -p gpurun_out
bash tools/r2_gpu_l.sh
echo "BIG" >> gpurun_out/l_red.log
for nm in "10000 20" "20000 50"; do
  set -- $nm
  SS_GEMM_BIG=1 timeout 300 python tools/red_probe.py --n $1 --m $2 --p $2 >> gpurun_out/l_red.log 2>&1
done
bash tools/r2_gpu_m.sh
