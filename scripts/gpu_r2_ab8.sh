# deferred tail with the wavefront's SMs reserved: tests + same-box A/B against the previous build
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_schedule.py -x -q > gpurun_out/pytest_ab8.log 2>&1; tail -2 gpurun_out/pytest_ab8.log
AB_REPS=3 AB_CFGS="SWTB_LIB=paper_2211_16270_b200/ab_base.so;SWTB_LIB=paper_2211_16270_b200/libswt_b200.so" timeout 1500 python scripts/gpu_ab.py
