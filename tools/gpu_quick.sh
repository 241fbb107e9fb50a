# Quick GPU iteration: two-level parity subset + config 2 / 4 timing.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "two_level or golden or medium or criterion4 or wide_m or config1" 2>&1 | tail -5 > gpurun_out/quick.log
timeout 300 python tools/diag.py --cfg 2 ${DIAG_ARGS} 2>&1 | grep -E "^cfg|shift 0:" >> gpurun_out/quick.log
timeout 300 python tools/diag.py --cfg 1 ${DIAG_ARGS} 2>&1 | grep -E "^cfg|shift 0:" >> gpurun_out/quick.log
timeout 600 python tools/diag.py --cfg 4 --reps 3 ${DIAG_ARGS} 2>&1 | grep -E "^cfg" >> gpurun_out/quick.log
cat gpurun_out/quick.log
