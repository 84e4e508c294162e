# round-2 evidence run: parity suite, c4 bench (both arms), C++ drop-in parity,
# ncu launch list + full capture of the hot kernels, compute-sanitizer
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1; tail -c 400 gpurun_out/bench_c4.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -c 1500 gpurun_out/bench_ref.log
timeout 900 ./oracle/_ref/ref_parity > gpurun_out/ref_parity.log 2>&1; tail -2 gpurun_out/ref_parity.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
  --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary \
  > gpurun_out/ncu_launch_bench.log 2>&1; tail -2 gpurun_out/ncu_launch_bench.log
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
  -k regex:'gemm_kernel|lattice|zslab|zmean|edge|reduce_partials' -c 24 \
  -o gpurun_out/prof_c4 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary \
  > gpurun_out/ncu_full_c4.log 2>&1; tail -2 gpurun_out/ncu_full_c4.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_case.py fp16,bf16 > gpurun_out/sanitize_$t.log 2>&1
  tail -3 gpurun_out/sanitize_$t.log
done
ls -la gpurun_out
