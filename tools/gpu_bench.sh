# Round-end style GPU run: tests, smoke, bench (both arms), ncu launch list of one
# bench step and one full ncu capture of the dominant kernel (k_far, mid sweep).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_k20.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_(block|far|seed|head|fro2|update|rq)' --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_launch.log 2>&1
python tools/far_traffic.py gpurun_out/launches.csv gpurun_out/far_traffic.json > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_far' -s 16 -c 2 -o gpurun_out/far_full --force-overwrite python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_block' -s 15 -c 1 -o gpurun_out/blk_full --force-overwrite python bench.py --profile --steps 1 --warmup 1 >> gpurun_out/ncu_full.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/bench_ref.log
