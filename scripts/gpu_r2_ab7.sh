# deferred group tail (ga/gl sums + joint backward between the next group's two backward parts): GPU suite + A/B against HEAD
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_ab7.log 2>&1; tail -2 gpurun_out/pytest_gpu_ab7.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu_ab7.log | head
timeout 900 ./oracle/_ref/ref_parity > gpurun_out/ref_parity.log 2>&1; tail -1 gpurun_out/ref_parity.log
AB_REPS=3 AB_CFGS="SWTB_LIB=paper_2211_16270_b200/ab_base.so;SWTB_LIB=paper_2211_16270_b200/libswt_b200.so" timeout 1500 python scripts/gpu_ab.py
