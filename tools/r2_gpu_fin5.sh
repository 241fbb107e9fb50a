#!/bin/bash
# Final product measurement pass (DFMA far kernels, suffix-product composites
# for every window-composite width incl. m = 1).
mkdir -p gpurun_out/f5
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f5/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/f5/pytest.log
timeout 900 python bench.py > gpurun_out/f5/bench4.log 2>&1
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f5/bench_ref.log 2>&1
for c in 1 2 3 5; do timeout 600 python bench.py --cfg $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/f5/bench$c.log 2>&1; done
for nm in "10000 20 2000" "20000 50 500" "4000 10 1000" "10000 1 2000"; do set -- $nm; timeout 300 python tools/lq_probe.py --n $1 --m $2 --s $3 >> gpurun_out/f5/lq.log 2>&1; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 4 2 3 5; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_ --csv --log-file gpurun_out/f5/launches_cfg$c.csv python bench.py --cfg $c --profile > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/f5/launches_cfg$c.csv > gpurun_out/f5/launch_sum_cfg$c.txt 2>&1
done
cp profiles/r2_far_traffic.json gpurun_out/f5/far_traffic.json
python tools/launch_traffic.py gpurun_out/f5/launches_cfg4.csv "k_fark<" 4 gpurun_out/f5/far_traffic.json > /dev/null 2>&1
python tools/launch_traffic.py gpurun_out/f5/launches_cfg2.csv "k_fark<" 2 gpurun_out/f5/far_traffic.json > /dev/null 2>&1
python tools/launch_traffic.py gpurun_out/f5/launches_cfg3.csv "k_farkm<" 3 gpurun_out/f5/far_traffic.json > /dev/null 2>&1
python tools/launch_traffic.py gpurun_out/f5/launches_cfg5.csv "k_fark<" 5 gpurun_out/f5/far_traffic.json > /dev/null 2>&1
F="--set full --clock-control none --import-source on"
timeout 600 ncu $F -k regex:k_fark --launch-skip 40 --launch-count 1 -o /tmp/f5_fk4 -f python bench.py --profile > /dev/null 2>&1
timeout 600 ncu $F -k regex:k_wsuffix --launch-skip 10 --launch-count 1 -o /tmp/f5_ws5 -f python bench.py --cfg 5 --profile > /dev/null 2>&1
python tools/ncu_summary.py - /tmp/f5_fk4.ncu-rep /tmp/f5_ws5.ncu-rep > gpurun_out/f5/ncu_full.txt 2>&1
echo done
