#!/bin/bash
# k_farkmd (m = 1 far pass / transposed w pass on DMMA): full suite + config 3 + transposed timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fm_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fm_pytest.log
timeout 600 python bench.py --cfg 3 --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > gpurun_out/fm_bench3.log 2>&1
FUZZ_NMAX=2500 timeout 400 python tools/fuzz_parity.py 13 16 > gpurun_out/fm_fuzz.log 2>&1
timeout 300 python tools/lq_probe.py --n 10000 --m 20 --s 2000 >> gpurun_out/fm_lq.jsonl 2>&1
timeout 300 python tools/lq_probe.py --n 10000 --m 1 --s 2000 >> gpurun_out/fm_lq.jsonl 2>&1
echo done
