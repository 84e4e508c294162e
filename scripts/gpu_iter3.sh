# full GPU suite + c4 bench (fp16 default, bf16 secondary) + group-size A/B
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
grep -E "c4 B'=8|c5 full" gpurun_out/pytest_gpu.log | cut -c1-200
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1; tail -c 400 gpurun_out/bench_c4.log
SWTB_GROUP_CELLS=524288 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/bench_c4_g19.log 2>&1
python scripts/bench_summary.py gpurun_out/bench_c4.log gpurun_out/bench_c4_g19.log
