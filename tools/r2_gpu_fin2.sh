#!/bin/bash
# Round-2 measurement pass after the DMMA far kernels (k_farkd / k_farkmd).
mkdir -p gpurun_out/f2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/f2/smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/f2/bench4.log 2>&1
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f2/bench_ref.log 2>&1
for c in 1 2 3 5; do timeout 600 python bench.py --cfg $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/f2/bench$c.log 2>&1; done
for nm in "10000 20 2000" "20000 50 500" "4000 10 1000" "10000 1 2000"; do set -- $nm; timeout 300 python tools/lq_probe.py --n $1 --m $2 --s $3 >> gpurun_out/f2/lq.log 2>&1; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 4 2 3 5; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_ --csv --log-file gpurun_out/f2/launches_cfg$c.csv python bench.py --cfg $c --profile > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/f2/launches_cfg$c.csv > gpurun_out/f2/launch_sum_cfg$c.txt 2>&1
done
cp profiles/r2_far_traffic.json gpurun_out/f2/far_traffic.json
python tools/launch_traffic.py gpurun_out/f2/launches_cfg4.csv k_farkd 4 gpurun_out/f2/far_traffic.json > /dev/null 2>&1
python tools/launch_traffic.py gpurun_out/f2/launches_cfg2.csv k_farkd 2 gpurun_out/f2/far_traffic.json > /dev/null 2>&1
python tools/launch_traffic.py gpurun_out/f2/launches_cfg3.csv k_farkmd 3 gpurun_out/f2/far_traffic.json > /dev/null 2>&1
python tools/launch_traffic.py gpurun_out/f2/launches_cfg5.csv k_farkd 5 gpurun_out/f2/far_traffic.json > /dev/null 2>&1
F="--set full --clock-control none --import-source on"
timeout 600 ncu $F -k regex:k_farkd --launch-skip 40 --launch-count 1 -o /tmp/f2_fk4 -f python bench.py --profile > /dev/null 2>&1
timeout 600 ncu $F -k regex:k_block --launch-skip 40 --launch-count 1 -o /tmp/f2_blk4 -f python bench.py --profile > /dev/null 2>&1
timeout 600 ncu $F -k regex:k_farkd --launch-skip 10 --launch-count 1 -o /tmp/f2_fk5 -f python bench.py --cfg 5 --profile > /dev/null 2>&1
timeout 600 ncu $F -k regex:k_farkmd --launch-skip 1 --launch-count 1 -o /tmp/f2_fkm3 -f python bench.py --cfg 3 --profile > /dev/null 2>&1
python tools/ncu_summary.py - /tmp/f2_fk4.ncu-rep /tmp/f2_blk4.ncu-rep /tmp/f2_fk5.ncu-rep /tmp/f2_fkm3.ncu-rep > gpurun_out/f2/ncu_full.txt 2>&1
for r in fk4 fk5 fkm3; do
  ncu -i /tmp/f2_$r.ncu-rep --page raw --csv > gpurun_out/f2/raw_$r.csv 2>/dev/null
done
echo done
