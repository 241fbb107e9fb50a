#!/bin/bash
# Round-2 final measurement pass: all configs, reference arm, ncu launch lists
# and full captures of every dominant kernel, reduction and transposed solve.
mkdir -p gpurun_out/v
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v/smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/v/bench4.log 2>&1
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/v/bench_ref.log 2>&1
for c in 1 2 3 5; do timeout 600 python bench.py --cfg $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/v/bench$c.log 2>&1; done
for nm in "2000 1" "4000 10" "10000 20" "20000 50"; do set -- $nm; timeout 300 python tools/red_probe.py --n $1 --m $2 --p $2 >> gpurun_out/v/red.log 2>&1; done
for nm in "10000 20 40" "20000 50 40" "4000 10 200"; do set -- $nm; timeout 300 python tools/lq_probe.py --n $1 --m $2 --s $3 >> gpurun_out/v/lq.log 2>&1; done
timeout 300 python tools/gemm_probe.py > gpurun_out/v/gemm.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
for c in 4 2 3 5; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:k_ --csv --log-file gpurun_out/v/launches_cfg$c.csv python bench.py --cfg $c --profile > /dev/null 2>&1
done
python tools/launch_traffic.py gpurun_out/v/launches_cfg4.csv k_fark 4 gpurun_out/v/far_traffic.json > /dev/null 2>&1
python tools/launch_traffic.py gpurun_out/v/launches_cfg5.csv k_fark 5 gpurun_out/v/far_traffic.json > /dev/null 2>&1
python tools/launch_traffic.py gpurun_out/v/launches_cfg3.csv k_farkm 3 gpurun_out/v/far_traffic.json > /dev/null 2>&1
python tools/launch_traffic.py gpurun_out/v/launches_cfg2.csv k_fark 2 gpurun_out/v/far_traffic.json > /dev/null 2>&1
F="--set full --clock-control none --import-source on"
timeout 600 ncu $F -k regex:k_fark --launch-skip 20 --launch-count 1 -o /tmp/v_fark4 -f python bench.py --profile > /dev/null 2>&1
timeout 600 ncu $F -k regex:k_block --launch-skip 20 --launch-count 1 -o /tmp/v_blk4 -f python bench.py --profile > /dev/null 2>&1
timeout 600 ncu $F -k regex:k_fark --launch-skip 10 --launch-count 1 -o /tmp/v_fark5 -f python bench.py --cfg 5 --profile > /dev/null 2>&1
timeout 600 ncu $F -k regex:k_rq_big --launch-skip 20 --launch-count 1 -o /tmp/v_rqbig5 -f python bench.py --cfg 5 --profile > /dev/null 2>&1
timeout 600 ncu $F -k regex:k_farkm --launch-skip 5 --launch-count 1 -o /tmp/v_farkm3 -f python bench.py --cfg 3 --profile > /dev/null 2>&1
timeout 600 ncu $F -k regex:k_rq_m1 --launch-skip 5 --launch-count 1 -o /tmp/v_rqm1 -f python bench.py --cfg 3 --profile > /dev/null 2>&1
timeout 600 ncu $F -k regex:"k_panel|k_dmma" --launch-skip 800 --launch-count 6 -o /tmp/v_red -f python tools/red_probe.py --n 10000 --m 20 --p 20 --profile > /dev/null 2>&1
timeout 600 ncu $F -k regex:"k_lq|k_tupd" --launch-skip 40 --launch-count 2 -o /tmp/v_lq -f python tools/lq_probe.py --n 10000 --m 20 --s 40 --profile > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 2000 --launch-count 400 --csv --log-file gpurun_out/v/launches_red10k.csv python tools/red_probe.py --n 10000 --m 20 --p 20 --profile > /dev/null 2>&1
for r in fark4 blk4 fark5 rqbig5 farkm3 rqm1 red lq; do
  python tools/ncu_summary.py - /tmp/v_$r.ncu-rep > gpurun_out/v/ncu_$r.txt 2>&1
done
for c in 4 2 3 5; do python tools/ncu_summary.py gpurun_out/v/launches_cfg$c.csv > gpurun_out/v/launch_sum_cfg$c.txt 2>&1; done
python tools/ncu_summary.py gpurun_out/v/launches_red10k.csv > gpurun_out/v/launch_sum_red10k.txt 2>&1
du -sh gpurun_out
