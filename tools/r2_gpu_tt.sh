#!/bin/bash
# transposed tail from the top block (k_ttail_s)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_transposed.py tests/test_gpu_irka.py -x -q > gpurun_out/tt_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/tt_pytest.log
for a in "--n 10000 --m 20 --s 2000" "--n 20000 --m 50 --s 500" "--n 4000 --m 10 --s 1000" "--n 10000 --m 29 --s 1000" "--n 10000 --m 1 --s 2000"; do
  timeout 300 python tools/lq_probe.py $a >> gpurun_out/tt_lq.jsonl 2>&1
done
FUZZ_NMAX=2500 timeout 400 python tools/fuzz_parity.py 43 12 > gpurun_out/tt_fuzz.log 2>&1
echo done
