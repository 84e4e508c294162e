# ncu evidence: launch list of one timed c4 step + full capture of each hot kernel (c3 step)
set -x
mkdir -p gpurun_out
# one c4 step after 3 warm-up steps (2531 launches/step at c4; skip the warm-ups)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 7600 -c 2600 --csv \
  --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_launch_bench.log 2>&1
# full sets: every distinct hot kernel once (c3: 4 groups/step)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gemm_kernel|lattice_kernel|zslab|split_rows' \
  -s 40 -c 12 -o gpurun_out/prof_c3 python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
