mkdir -p gpurun_out
python tools/diag.py --variants "SS_STREAMS=1" > gpurun_out/diag17.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest17.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_block' -s 15 -c 1 -o gpurun_out/blk17 --force-overwrite python tools/diag.py --profile > gpurun_out/ncu_full17.log 2>&1
cat gpurun_out/diag17.log gpurun_out/pytest17.log
