#!/bin/bash
# Round-2 GPU pass A: build check, full GPU test suite (incl. full-size configs),
# config-4 bench + reference arm, ncu launch list and full captures of the
# config-4 sweep kernels.  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/a_pytest.log
timeout 600 python bench.py > gpurun_out/a_bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/a_bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:k_ --csv --log-file gpurun_out/a_launches_cfg4.csv \
  python bench.py --profile --steps 1 --warmup 0 > gpurun_out/a_ncu_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_far --launch-skip 40 --launch-count 1 \
  -o gpurun_out/a_far_cfg4 -f python bench.py --profile > gpurun_out/a_ncu_far.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_block --launch-skip 20 --launch-count 1 \
  -o gpurun_out/a_blk_cfg4 -f python bench.py --profile > gpurun_out/a_ncu_blk.log 2>&1
echo done
