# round-2 iteration: full GPU suite + c4 bench (fp16 default) + A/B knobs
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
grep -E "c4 B'=8|c5 full" gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_fp16.log 2>&1; tail -c 300 gpurun_out/bench_c4_fp16.log
SWTB_FWD_CORR=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_fp16_nocorr.log 2>&1; tail -c 300 gpurun_out/bench_c4_fp16_nocorr.log
python scripts/bench_summary.py gpurun_out/bench_c4_fp16.log gpurun_out/bench_c4_fp16_nocorr.log 2>&1 | tail -20
