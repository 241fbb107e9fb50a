# usage: bash tools/gpu_diag.sh  (on the GPU box)
mkdir -p gpurun_out
python tools/diag.py --variants "SS_STREAMS=1,SS_STREAMS=2,SS_STREAMS=1;SS_UPDATE_CLASSIC=1,SS_STREAMS=2;SS_UPDATE_CLASSIC=1,SS_STREAMS=1;SS_BLOCK_RQ=givens" > gpurun_out/diag.log 2>&1
SS_STREAMS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_update|k_rq_house' -s 60 -c 2 -o gpurun_out/upd_rq --force-overwrite python tools/diag.py --profile > gpurun_out/ncu_full.log 2>&1
SS_STREAMS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(update|rq|head|seed|fro2)' --csv --log-file gpurun_out/launches_sweep.csv python tools/diag.py --profile > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/diag.log
