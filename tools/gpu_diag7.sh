mkdir -p gpurun_out
for v in s8m4 s6m4 s5m4 s6m5; do echo "== $v"; SS_LIB_PATH=$PWD/build_var/lib_$v.so python tools/diag.py --variants "SS_STREAMS=1,SS_STREAMS=2" 2>&1 | grep cfg2; done > gpurun_out/diag7.log 2>&1
cat gpurun_out/diag7.log
