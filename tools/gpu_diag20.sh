mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv > gpurun_out/diag20.log
timeout 200 python tools/diag.py --variants "SS_STREAMS=1,SS_FAR_NST7=1" >> gpurun_out/diag20.log 2>&1
SS_LIB_PATH=$PWD/build_var/lib_far128.so timeout 200 python tools/diag.py --variants "SS_STREAMS=1,SS_FAR_NST7=1" >> gpurun_out/diag20.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv >> gpurun_out/diag20.log
cat gpurun_out/diag20.log
