mkdir -p gpurun_out
timeout 600 python tools/diag.py --cfg 4 --reps 3 --variants "SS_STREAMS=1,SS_UPDATE_CLASSIC=1;SS_STREAMS=2" 2>&1 | grep -E "^cfg|rror" > gpurun_out/diag24.log
timeout 600 python -m pytest tests -m gpu -x -q -k "wide_m or medium or two_level" 2>&1 | tail -3 >> gpurun_out/diag24.log
cat gpurun_out/diag24.log
