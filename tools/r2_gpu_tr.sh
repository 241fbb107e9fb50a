#!/bin/bash
# transposed sweep on k_farkd: parity + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_transposed.py tests/test_gpu_irka.py -x -q > gpurun_out/tr_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/tr_pytest.log
FUZZ_NMAX=2500 timeout 400 python tools/fuzz_parity.py 11 16 > gpurun_out/tr_fuzz.log 2>&1
for a in "--n 10000 --m 20 --s 2000" "--n 20000 --m 50 --s 500" "--n 4000 --m 10 --s 1000" "--n 10000 --m 29 --s 1000" "--n 10000 --m 40 --s 500"; do
  timeout 300 python tools/lq_probe.py $a >> gpurun_out/tr_lq.jsonl 2>&1
done
echo done
