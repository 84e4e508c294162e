# Round evidence: parity suites, the default bench line (with e2e + CPU
# baseline), the reference arm, an ncu launch list of one timed c4 step and a
# full ncu capture of the hot kernels of a c4 step.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 ./oracle/_ref/ref_parity > gpurun_out/ref_parity.log 2>&1; tail -1 gpurun_out/ref_parity.log
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 400 gpurun_out/bench_default.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>&1; tail -c 300 gpurun_out/bench_reference.json
# launch list: the timed c4 step (NVTX range "timed" of bench.py) after 3 warm-up steps
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
  --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_launch_bench.log 2>&1
# full capture: the hot kernels of the first c4 groups (after warm-up)
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
  -k regex:'gemm_kernel|lattice|zslab|edge|reduce_partials|split_rows' -c 16 \
  -o gpurun_out/prof_c4 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_full_c4.log 2>&1; tail -2 gpurun_out/ncu_full_c4.log
ls -la gpurun_out
