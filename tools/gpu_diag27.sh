mkdir -p gpurun_out
timeout 600 python tools/diag.py --cfg 4 --reps 3 --variants "SS_STREAMS=1,SS_ONE_LEVEL=1" 2>&1 | grep -E "^cfg|rror" > gpurun_out/diag27.log
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 >> gpurun_out/diag27.log
cat gpurun_out/diag27.log
