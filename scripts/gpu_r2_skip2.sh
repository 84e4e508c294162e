# zero-tile skip: full GPU suite, C++ parity, bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_skip.log 2>&1; tail -2 gpurun_out/pytest_skip.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_skip.log | head -10
grep -E "c4 B'=8|c5 full" gpurun_out/pytest_skip.log | cut -c1-200
timeout 900 ./oracle/_ref/ref_parity > gpurun_out/ref_parity.log 2>&1; tail -1 gpurun_out/ref_parity.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_skip.json 2>gpurun_out/bench_skip.err; python scripts/bench_summary.py gpurun_out/bench_skip.json; tail -3 gpurun_out/bench_skip.err
