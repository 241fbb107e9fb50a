#!/bin/bash
# Round-2 GPU pass I: reduction timing at scale, configs 2/3/5 bench lines,
# ncu launch lists + full captures of the config-5 / config-3 kernels, the
# reduction's kernels and the transposed solver's.
mkdir -p gpurun_out
for nm in "4000 10" "10000 20" "20000 50" "2000 1"; do
  set -- $nm
  timeout 300 python tools/red_probe.py --n $1 --m $2 --p $2 >> gpurun_out/i_red.log 2>&1
done
timeout 600 python bench.py --cfg 5 --no-cpu-baseline --no-e2e --steps 3 --warmup 1 > gpurun_out/i_bench5.log 2>&1
timeout 300 python bench.py --cfg 3 --no-cpu-baseline --no-e2e > gpurun_out/i_bench3.log 2>&1
timeout 300 python bench.py --cfg 2 --no-cpu-baseline --no-e2e > gpurun_out/i_bench2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:k_ --csv --log-file gpurun_out/i_launches_cfg5.csv \
  python bench.py --cfg 5 --profile > gpurun_out/i_ncu_list5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:k_ --csv --log-file gpurun_out/i_launches_cfg3.csv \
  python bench.py --cfg 3 --profile > gpurun_out/i_ncu_list3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum \
  --clock-control none --csv --log-file gpurun_out/i_launches_red.csv \
  python tools/red_probe.py --n 1500 --m 10 --p 10 --profile > gpurun_out/i_ncu_listred.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rq_big --launch-skip 20 --launch-count 1 \
  -o gpurun_out/i_rqbig_cfg5 -f python bench.py --cfg 5 --profile > gpurun_out/i_ncu_rqbig.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update --launch-skip 20 --launch-count 1 \
  -o gpurun_out/i_upd_cfg5 -f python bench.py --cfg 5 --profile > gpurun_out/i_ncu_upd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rq_m1 --launch-skip 10 --launch-count 1 \
  -o gpurun_out/i_rqm1_cfg3 -f python bench.py --cfg 3 --profile > gpurun_out/i_ncu_rqm1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_far --launch-skip 10 --launch-count 1 \
  -o gpurun_out/i_far_cfg3 -f python bench.py --cfg 3 --profile > gpurun_out/i_ncu_far3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dgemm --launch-skip 300 --launch-count 2 \
  -o gpurun_out/i_dgemm -f python tools/red_probe.py --n 4000 --m 10 --p 10 --profile > gpurun_out/i_ncu_dgemm.log 2>&1

# summaries on the box; the full reports stay there (gpurun_out is capped at 64 MiB)
python tools/ncu_summary.py gpurun_out/i_launches_cfg5.csv gpurun_out/i_rqbig_cfg5.ncu-rep gpurun_out/i_upd_cfg5.ncu-rep > gpurun_out/i_sum_cfg5.txt 2>&1
python tools/ncu_summary.py gpurun_out/i_launches_cfg3.csv gpurun_out/i_rqm1_cfg3.ncu-rep gpurun_out/i_far_cfg3.ncu-rep > gpurun_out/i_sum_cfg3.txt 2>&1
python tools/ncu_summary.py gpurun_out/i_launches_red.csv gpurun_out/i_dgemm.ncu-rep > gpurun_out/i_sum_red.txt 2>&1
mkdir -p /tmp/reps; mv gpurun_out/*.ncu-rep /tmp/reps/ 2>/dev/null
du -sh gpurun_out
