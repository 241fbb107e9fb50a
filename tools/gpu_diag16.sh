mkdir -p gpurun_out
for c in 1 3; do timeout 300 python tools/diag.py --cfg $c --reps 3; done > gpurun_out/diag16.log 2>&1
timeout 300 python tools/diag.py --cfg 4 --reps 2 --shifts 2000 >> gpurun_out/diag16.log 2>&1
timeout 600 python tools/diag.py --cfg 5 --reps 1 --shifts 500 >> gpurun_out/diag16.log 2>&1
cat gpurun_out/diag16.log
