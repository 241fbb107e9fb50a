mkdir -p gpurun_out
python tools/diag.py --variants "SS_STREAMS=1" > gpurun_out/diag14.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_far' -s 30 -c 2 -o gpurun_out/far14 --force-overwrite python tools/diag.py --profile > gpurun_out/ncu_full14.log 2>&1
cat gpurun_out/diag14.log
