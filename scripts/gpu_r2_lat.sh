# wavefront warps per (sample, direction) after the zero-tile skip: 2 / 4 (default at c4) / 8
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
AB_REPS=2 AB_CFGS="SWTB_LAT_W=4;SWTB_LAT_W=2;SWTB_LAT_W=8" timeout 1800 python scripts/gpu_ab.py
