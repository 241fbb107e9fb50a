mkdir -p gpurun_out
timeout 300 python tools/diag.py --cfg 3 --variants "SS_STREAMS=1,SS_NO_MSH=1" 2>&1 | grep -E "^cfg|shift|rror" > gpurun_out/diag25.log
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 >> gpurun_out/diag25.log
cat gpurun_out/diag25.log
