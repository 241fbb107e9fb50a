mkdir -p gpurun_out
python tools/diag.py --variants "SS_STREAMS=1,SS_STREAMS=2,SS_STREAMS=1;SS_ONE_LEVEL=1" > gpurun_out/diag4.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest4.log
SS_STREAMS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_update_ws|k_block' -s 20 -c 3 -o gpurun_out/blk4 --force-overwrite python tools/diag.py --profile > gpurun_out/ncu_full4.log 2>&1
cat gpurun_out/diag4.log gpurun_out/pytest4.log
