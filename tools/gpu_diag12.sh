mkdir -p gpurun_out
python tools/diag.py --variants "SS_STREAMS=1,SS_STREAMS=1;SS_FAR_SPIN=1,SS_STREAMS=1;SS_FAR_JH=2,SS_STREAMS=1;SS_FAR_JH=-2,SS_STREAMS=1;SS_FAR_JH=4" > gpurun_out/diag12.log 2>&1
cat gpurun_out/diag12.log
