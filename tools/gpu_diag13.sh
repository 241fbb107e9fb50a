mkdir -p gpurun_out
python tools/diag.py --variants "SS_STREAMS=1,SS_STREAMS=1;SS_FAR_R4=1" > gpurun_out/diag13.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest13.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_far' -s 20 -c 2 -o gpurun_out/far13 --force-overwrite python tools/diag.py --profile > gpurun_out/ncu_full13.log 2>&1
cat gpurun_out/diag13.log gpurun_out/pytest13.log
