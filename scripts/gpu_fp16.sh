# fp16 mode bring-up: parity (c1..c5 subsets) + c4 bench
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_step.py -x -q -s -k "fp16 or c4_subset or c5_full" > gpurun_out/pytest_fp16.log 2>&1; tail -30 gpurun_out/pytest_fp16.log
timeout 600 python bench.py --steps 3 --warmup 3 --precision fp16 --no-cpu-baseline > gpurun_out/bench_c4_fp16.log 2>&1; tail -c 1500 gpurun_out/bench_c4_fp16.log
