#!/bin/bash
mkdir -p gpurun_out
for s in VtM MV rank64_NT; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_dmma -c 1 \
  -o gpurun_out/q_$s -f python tools/gemm_probe.py $s > gpurun_out/q_ncu_$s.log 2>&1
done
python tools/ncu_summary.py - gpurun_out/q_VtM.ncu-rep gpurun_out/q_MV.ncu-rep gpurun_out/q_rank64_NT.ncu-rep > gpurun_out/q_sum.txt 2>&1
