# last check of HEAD: smoke, full GPU suite, C++ parity
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_last.log 2>&1; tail -1 gpurun_out/pytest_gpu_last.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu_last.log | head
timeout 900 ./oracle/_ref/ref_parity > gpurun_out/ref_parity_last.log 2>&1; tail -1 gpurun_out/ref_parity_last.log
