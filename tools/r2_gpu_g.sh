#!/bin/bash
# Round-2 GPU pass G: full GPU suite, config-4 bench + reference arm,
# ncu launch list (+ per-launch DRAM), full captures of k_fark / k_block<20>.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/g_pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:k_ --csv --log-file gpurun_out/g_launches_cfg4.csv \
  python bench.py --profile > gpurun_out/g_ncu_list.log 2>&1
python tools/launch_traffic.py gpurun_out/g_launches_cfg4.csv k_fark 4 profiles/r2_far_traffic.json > gpurun_out/g_traffic.log 2>&1
timeout 900 python bench.py > gpurun_out/g_bench.log 2>&1
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g_bench_ref.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fark --launch-skip 6 --launch-count 1 \
  -o gpurun_out/g_fark_cfg4 -f python bench.py --profile > gpurun_out/g_ncu_fark.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_block --launch-skip 20 --launch-count 1 \
  -o gpurun_out/g_blk_cfg4 -f python bench.py --profile > gpurun_out/g_ncu_blk.log 2>&1
cp profiles/r2_far_traffic.json gpurun_out/ 2>/dev/null
echo done
