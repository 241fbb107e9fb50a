mkdir -p gpurun_out
: > gpurun_out/diag22.log
for c in 1 3; do timeout 200 python tools/diag.py --cfg $c --variants "SS_STREAMS=1,SS_ONE_LEVEL=1,SS_ONE_LEVEL=1;SS_STREAMS=1" 2>&1 | grep -E "cfg" >> gpurun_out/diag22.log; done
timeout 300 python tools/diag.py --cfg 4 --reps 3 --variants "SS_STREAMS=1,SS_STREAMS=2" 2>&1 | grep -E "cfg" >> gpurun_out/diag22.log
cat gpurun_out/diag22.log
