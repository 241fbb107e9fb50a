#!/bin/bash
# Round-2 final measurement pass (after the reduction / transposed work).
mkdir -p gpurun_out/f
timeout 900 python bench.py > gpurun_out/f/bench4.log 2>&1
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f/bench_ref.log 2>&1
for c in 1 2 3 5; do timeout 600 python bench.py --cfg $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/f/bench$c.log 2>&1; done
for nm in "2000 1" "4000 10" "10000 20" "20000 50"; do set -- $nm; timeout 300 python tools/red_probe.py --n $1 --m $2 --p $2 >> gpurun_out/f/red.log 2>&1; done
for nm in "10000 20 40" "10000 20 2000" "20000 50 500" "4000 10 1000"; do set -- $nm; timeout 300 python tools/lq_probe.py --n $1 --m $2 --s $3 >> gpurun_out/f/lq.log 2>&1; done
timeout 300 python tools/gemm_probe.py > gpurun_out/f/gemm.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:k_ --csv --log-file gpurun_out/f/launches_cfg4.csv python bench.py --profile > /dev/null 2>&1
python tools/launch_traffic.py gpurun_out/f/launches_cfg4.csv k_fark 4 gpurun_out/f/far_traffic.json > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 1000 --launch-count 500 --csv --log-file gpurun_out/f/launches_red10k.csv python tools/red_probe.py --n 10000 --m 20 --p 20 --profile > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/f/launches_tr.csv python tools/lq_probe.py --n 10000 --m 20 --s 2000 --profile > /dev/null 2>&1
F="--set full --clock-control none --import-source on"
timeout 600 ncu $F -k regex:k_panel --launch-skip 100 --launch-count 1 -o /tmp/f_panel -f python tools/red_probe.py --n 10000 --m 20 --p 20 --profile > /dev/null 2>&1
timeout 600 ncu $F -k regex:k_dmma --launch-skip 600 --launch-count 4 -o /tmp/f_dmma -f python tools/red_probe.py --n 10000 --m 20 --p 20 --profile > /dev/null 2>&1
timeout 600 ncu $F -k regex:"k_fark|k_tr_lower|k_lq" --launch-skip 30 --launch-count 3 -o /tmp/f_tr -f python tools/lq_probe.py --n 10000 --m 20 --s 2000 --profile > /dev/null 2>&1
for r in panel dmma tr; do python tools/ncu_summary.py - /tmp/f_$r.ncu-rep > gpurun_out/f/ncu_$r.txt 2>&1; done
for x in cfg4 red10k tr; do python tools/ncu_summary.py gpurun_out/f/launches_$x.csv > gpurun_out/f/launch_sum_$x.txt 2>&1; done
