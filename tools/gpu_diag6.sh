mkdir -p gpurun_out
python tools/diag.py --variants "SS_STREAMS=1,SS_STREAMS=2" > gpurun_out/diag6.log 2>&1
SS_LIB_PATH=$PWD/build_var/lib_mb4.so python tools/diag.py --variants "SS_STREAMS=1,SS_STREAMS=2" >> gpurun_out/diag6.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest6.log
SS_STREAMS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_block' -s 10 -c 1 -o gpurun_out/blk6 --force-overwrite python tools/diag.py --profile > gpurun_out/ncu_full6.log 2>&1
cat gpurun_out/diag6.log gpurun_out/pytest6.log
