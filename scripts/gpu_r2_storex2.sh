# stored logits: double-buffered staging, dh beside the GEMMs; same-box A/B
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 900 python -m pytest tests/test_gpu_schedule.py -x -q -s -k "store_x" > gpurun_out/pytest_storex.log 2>&1; tail -3 gpurun_out/pytest_storex.log
for r in 1 2; do
for cfg in "SWTB_STORE_X=1" "SWTB_STORE_X=1 SWTB_X2DH_SIDE=0" "SWTB_STORE_X=0"; do
  tag=$(echo $cfg | tr ' =' '_-')
  env $cfg timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/bench_$tag.$r.log 2>&1
  echo "$cfg"; python scripts/bench_summary.py gpurun_out/bench_$tag.$r.log
done
done
