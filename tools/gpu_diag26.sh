mkdir -p gpurun_out
timeout 300 python tools/diag.py --cfg 3 2>&1 | grep -E "^cfg|rror" > gpurun_out/diag26.log
timeout 300 python tools/diag.py --cfg 2 --variants "SS_ONE_LEVEL=1;SS_STREAMS=1" 2>&1 | grep -E "^cfg|rror" >> gpurun_out/diag26.log
timeout 300 python tools/diag.py --cfg 4 --reps 2 2>&1 | grep -E "^cfg|rror" >> gpurun_out/diag26.log
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/diag26.log
cat gpurun_out/diag26.log
