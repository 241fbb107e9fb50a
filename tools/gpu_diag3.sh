mkdir -p gpurun_out
python tools/diag.py --variants "SS_STREAMS=1;SS_WS_KW=3,SS_STREAMS=1;SS_WS_KW=2,SS_STREAMS=1;SS_WS_KW=1,SS_STREAMS=2;SS_WS_KW=3" > gpurun_out/diag3.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest3.log
SS_STREAMS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_update_ws' -s 30 -c 1 -o gpurun_out/upd3 --force-overwrite python tools/diag.py --profile > gpurun_out/ncu_full3.log 2>&1
cat gpurun_out/diag3.log gpurun_out/pytest3.log
