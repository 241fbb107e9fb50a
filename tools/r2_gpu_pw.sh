#!/bin/bash
# k_farkd with the in-warp producer (8 warps) for m = 40 / 50 / 60
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_transposed.py -x -q -k "wide or config5 or golden or transposed" > gpurun_out/pw_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pw_pytest.log
timeout 600 python bench.py --cfg 5 --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > gpurun_out/pw_bench5.log 2>&1
for a in "--n 20000 --m 50 --s 500" "--n 10000 --m 40 --s 500" "--n 10000 --m 59 --s 500"; do
  timeout 300 python tools/lq_probe.py $a >> gpurun_out/pw_lq.jsonl 2>&1
done
FUZZ_NMAX=2500 timeout 500 python tools/fuzz_parity.py 21 12 > gpurun_out/pw_fuzz.log 2>&1
echo done
