# store_x (dh from the forward's stored fp16 logits) vs recompute: parity + same-box A/B
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 900 python -m pytest tests/test_gpu_schedule.py tests/test_gpu_step.py -x -q -s > gpurun_out/pytest_storex.log 2>&1; tail -3 gpurun_out/pytest_storex.log
for r in 1 2; do
for x in 1 0; do
  SWTB_STORE_X=$x timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/bench_x$x.$r.log 2>&1
  python scripts/bench_summary.py gpurun_out/bench_x$x.$r.log
done
done
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_case.py fp16 > gpurun_out/sanitize_racecheck2.log 2>&1
tail -3 gpurun_out/sanitize_racecheck2.log; grep -c "Error:" gpurun_out/sanitize_racecheck2.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_case.py fp16,bf16 > gpurun_out/sanitize_memcheck2.log 2>&1
tail -2 gpurun_out/sanitize_memcheck2.log
