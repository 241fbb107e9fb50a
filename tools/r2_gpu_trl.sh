#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/trl_launches.csv python tools/lq_probe.py --n 10000 --m 20 --s 2000 --profile > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/trl_launches.csv > gpurun_out/trl_sum.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/trl_irka.csv python -c "
import sys; sys.argv=['bench.py','--profile']
" > /dev/null 2>&1
echo done
