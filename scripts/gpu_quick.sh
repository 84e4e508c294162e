# parity suite + c4 bench line + C++ drop-in parity driver
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 ./oracle/_ref/ref_parity > gpurun_out/ref_parity.log 2>&1; tail -2 gpurun_out/ref_parity.log
timeout 900 python bench.py --steps 3 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_c4.log 2>&1; tail -c 1500 gpurun_out/bench_c4.log
