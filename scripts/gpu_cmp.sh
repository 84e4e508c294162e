# parity suite + C++ parity + c4 bench per cluster size
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 ./oracle/_ref/ref_parity --quick > gpurun_out/ref_parity.log 2>&1; tail -1 gpurun_out/ref_parity.log
for cs in ${CS_LIST:-2}; do
  SWTB_CTA_GROUP=$cs timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_cs$cs.log 2>&1
  python scripts/bench_summary.py gpurun_out/bench_c4_cs$cs.log
done
