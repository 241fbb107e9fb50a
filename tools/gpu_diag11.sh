mkdir -p gpurun_out
python tools/diag.py --variants "SS_STREAMS=1,SS_STREAMS=2" > gpurun_out/diag11.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest11.log
SS_STREAMS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_block' -s 10 -c 1 -o gpurun_out/blk11 --force-overwrite python tools/diag.py --profile > gpurun_out/ncu_full11.log 2>&1
cat gpurun_out/diag11.log gpurun_out/pytest11.log
