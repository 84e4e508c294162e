# max-free forward log-sum-exp under the logit bound: tests + same-box A/B; group size / joint batch
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_ab6.log 2>&1; tail -2 gpurun_out/pytest_ab6.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_ab6.log | head
AB_REPS=2 AB_CFGS="SWTB_LIB=paper_2211_16270_b200/ab_base.so;SWTB_LIB=paper_2211_16270_b200/libswt_b200.so;SWTB_GROUP_CELLS=1572864 SWTB_JOINT_BATCH=6" timeout 1800 python scripts/gpu_ab.py
SWTB_GROUP_CELLS=1572864 SWTB_JOINT_BATCH=6 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline > gpurun_out/bench_g15.json 2>&1; python scripts/bench_summary.py gpurun_out/bench_g15.json | head -2
