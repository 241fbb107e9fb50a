mkdir -p gpurun_out
timeout 200 python tools/diag.py --variants "SS_STREAMS=1" 2>&1 > gpurun_out/diag19.log 2>&1
cat gpurun_out/diag19.log
