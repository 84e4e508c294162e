set -x
timeout 900 python -m pytest tests/test_gpu_modes.py -q > gpurun_out/pytest_modes.log 2>&1; tail -1 gpurun_out/pytest_modes.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_modes.log | head
SWTB_JOINT_BATCH=4 timeout 900 python -m pytest tests/test_gpu_modes.py -q -k memory_scaling > gpurun_out/pytest_modes4.log 2>&1; tail -1 gpurun_out/pytest_modes4.log
