# schedule knobs after the zero-tile skip: lead-part share, parts, group size
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
AB_REPS=2 AB_CFGS="SWTB_LEAD=0.25;SWTB_LEAD=0.35;SWTB_LEAD=0.18;SWTB_PARTS=3;SWTB_GROUP_CELLS=1572864;SWTB_JOINT_BATCH=8" timeout 2400 python scripts/gpu_ab.py
