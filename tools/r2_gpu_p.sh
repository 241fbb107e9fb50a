#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:k_dmma --launch-skip 2000 --launch-count 12 \
  -o gpurun_out/p_gemm -f python tools/red_probe.py --n 20000 --m 50 --p 50 --profile > gpurun_out/p_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_panel --launch-skip 200 --launch-count 1 \
  -o gpurun_out/p_panel -f python tools/red_probe.py --n 20000 --m 50 --p 50 --profile > gpurun_out/p_ncu2.log 2>&1
python tools/ncu_summary.py gpurun_out/p_gemm.ncu-rep gpurun_out/p_panel.ncu-rep > gpurun_out/p_sum.txt 2>&1
ncu -i gpurun_out/p_gemm.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,launch__grid_size,sm__inst_executed_pipe_fp64.sum,smsp__sass_thread_inst_executed_op_dmma_pred_on.sum,sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active > gpurun_out/p_gemm_raw.csv 2>&1
rm -f gpurun_out/*.ncu-rep
