mkdir -p gpurun_out
timeout 120 python tools/diag.py --variants "SS_STREAMS=1,SS_BLOCK_1W=1" > gpurun_out/diag18.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest18.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:'k_block' -s 15 -c 1 -o gpurun_out/blk18 --force-overwrite python tools/diag.py --profile > gpurun_out/ncu_full18.log 2>&1
cat gpurun_out/diag18.log gpurun_out/pytest18.log
