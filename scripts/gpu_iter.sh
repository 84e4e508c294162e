# iteration: parity suite, c4 bench line, ncu full capture of the hot kernels on a c3 step
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_c4.log 2>&1; tail -c 300 gpurun_out/bench_c4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gemm_kernel|lattice|zslab|edge' \
  -s 40 -c ${NCU_COUNT:-10} -o gpurun_out/prof_iter -f python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_iter.log 2>&1; tail -2 gpurun_out/ncu_iter.log
