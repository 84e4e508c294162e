# round-2 baseline: GPU parity suite, c4 bench lines in each precision mode
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for p in bf16 bf16x tf32; do
  timeout 600 python bench.py --steps 3 --warmup 3 --precision $p --no-cpu-baseline > gpurun_out/bench_c4_$p.log 2>&1
  tail -c 600 gpurun_out/bench_c4_$p.log
done
