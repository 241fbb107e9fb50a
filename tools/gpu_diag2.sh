mkdir -p gpurun_out
python tools/diag.py --variants "SS_STREAMS=1,SS_STREAMS=2,SS_STREAMS=2;SS_WS_STAGES=7,SS_STREAMS=2;SS_WS_STAGES=6,SS_STREAMS=2;SS_WS_STAGES=5,SS_STREAMS=1;SS_WS_STAGES=5" > gpurun_out/diag2.log 2>&1
SS_STREAMS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_update_ws' -s 30 -c 1 -o gpurun_out/upd2 --force-overwrite python tools/diag.py --profile > gpurun_out/ncu_full2.log 2>&1
cat gpurun_out/diag2.log
