# wavefront rows per lane: 2 (default) vs 1 (7 warps at U1 = 201)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_lat2.log 2>&1; tail -1 gpurun_out/pytest_lat2.log
SWTB_LAT_R=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_lat2r1.log 2>&1; tail -1 gpurun_out/pytest_lat2r1.log
AB_REPS=3 AB_CFGS="SWTB_LAT_R=2;SWTB_LAT_R=1" timeout 1800 python scripts/gpu_ab.py
