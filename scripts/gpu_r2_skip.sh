# zero-tile skip: GPU suite + same-build A/B (skip on / off)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_skip.log 2>&1; tail -2 gpurun_out/pytest_skip.log; grep -E "FAIL|Error" gpurun_out/pytest_skip.log | head -5
AB_REPS=2 AB_CFGS="SWTB_SKIP_ZERO_TILES=0;SWTB_SKIP_ZERO_TILES=1" timeout 1500 python scripts/gpu_ab.py
