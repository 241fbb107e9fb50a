# Per-config throughput on one B200 (tools/diag.py: synthetic m-Hessenberg triple
# of the config shape, ss_tf_eval, median of per-call CUDA-event times).
mkdir -p gpurun_out
: > gpurun_out/configs.log
for c in 1 2 3; do timeout 300 python tools/diag.py --cfg $c 2>&1 | grep -E "^cfg|shift 0:" >> gpurun_out/configs.log; done
timeout 600 python tools/diag.py --cfg 4 --reps 3 2>&1 | grep -E "^cfg|shift" >> gpurun_out/configs.log
timeout 900 python tools/diag.py --cfg 5 --reps 1 --shifts 500 2>&1 | grep -E "^cfg|shift" >> gpurun_out/configs.log
cat gpurun_out/configs.log
