# wavefront overlap after the tighter zero-tile bound: lead-part share / parts
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
AB_REPS=2 AB_CFGS="SWTB_LEAD=0.25;SWTB_LEAD=0.33;SWTB_LEAD=0.4;SWTB_PARTS=3;SWTB_PARTS=3 SWTB_LEAD=0.4" timeout 2400 python scripts/gpu_ab.py
