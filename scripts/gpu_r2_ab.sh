# same-box A/B of two builds (SWTB_LIB)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
AB_REPS=3 AB_CFGS="SWTB_LIB=paper_2211_16270_b200/ab_base.so;SWTB_LIB=paper_2211_16270_b200/libswt_b200.so" timeout 1500 python scripts/gpu_ab.py
