# lead part share with the deferred tail
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
AB_REPS=2 AB_CFGS="SWTB_LEAD=0.3;SWTB_LEAD=0.35;SWTB_LEAD=0.4;SWTB_LEAD=0.45" timeout 1800 python scripts/gpu_ab.py
