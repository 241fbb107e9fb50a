mkdir -p gpurun_out
timeout 300 python tools/diag.py --variants "SS_STREAMS=1,SS_FAR_P3=1" 2>&1 | grep -E "cfg2|shift 500|rror" > gpurun_out/diag23.log
cat gpurun_out/diag23.log
