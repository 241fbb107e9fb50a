#!/bin/bash
# forward wide-window composites built by the suffix product: parity + cfg5/cfg3 timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "wide or golden or medium or streamed or pseudo or config5 or config3" > gpurun_out/z_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/z_pytest.log
timeout 900 python -m pytest tests/test_gpu_transposed.py -x -q >> gpurun_out/z_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/z_pytest.log
timeout 600 python bench.py --cfg 5 --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > gpurun_out/z_bench5.log 2>&1
timeout 600 python bench.py --cfg 3 --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > gpurun_out/z_bench3.log 2>&1
echo done
for a in "--n 10000 --m 20 --s 2000" "--n 20000 --m 50 --s 500"; do
  timeout 300 python tools/lq_probe.py $a >> gpurun_out/z_lq.jsonl 2>&1
done
