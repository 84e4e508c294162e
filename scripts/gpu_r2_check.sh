# final check: driver-style build products present, smoke(), fixed schedule test, short bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_schedule.py -x -q > gpurun_out/pytest_check.log 2>&1; tail -2 gpurun_out/pytest_check.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_check.json 2>&1; python scripts/bench_summary.py gpurun_out/bench_check.json | head -2
