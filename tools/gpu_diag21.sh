mkdir -p gpurun_out
: > gpurun_out/diag21.log
for v in base u11 u11r6 u22; do
  if [ $v = base ]; then lib=""; else lib=$PWD/build_var/lib_$v.so; fi
  echo "== $v" >> gpurun_out/diag21.log
  SS_LIB_PATH=$lib timeout 200 python tools/diag.py 2>&1 | grep -E "cfg2|shift 500|Error" >> gpurun_out/diag21.log
done
cat gpurun_out/diag21.log
