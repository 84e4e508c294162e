# GPU suite after the last kernel edit; lead part 0.4 vs 0.5
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_t3.log 2>&1; tail -2 gpurun_out/pytest_gpu_t3.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu_t3.log | head
AB_REPS=2 AB_CFGS="SWTB_LEAD=0.4;SWTB_LEAD=0.5" timeout 1200 python scripts/gpu_ab.py
