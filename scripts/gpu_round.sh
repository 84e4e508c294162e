set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_c2.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.log 2>&1
tail -3 gpurun_out/pytest_gpu.log gpurun_out/bench_c2.log gpurun_out/bench_c4.log
