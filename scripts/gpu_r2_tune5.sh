# joint-network batch size with the deferred tail
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
AB_REPS=3 AB_CFGS="SWTB_JOINT_BATCH=4;SWTB_JOINT_BATCH=8" timeout 1800 python scripts/gpu_ab.py
SWTB_JOINT_BATCH=8 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline > gpurun_out/bench_jb8.json 2>&1; python scripts/bench_summary.py gpurun_out/bench_jb8.json | head -1
