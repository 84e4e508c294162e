# lattice kernel deep-dive: ncu source-level capture of two c4 launches
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'lattice' -s 20 -c 2 \
  -o gpurun_out/prof_lat -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_lat.log 2>&1
tail -2 gpurun_out/ncu_lat.log
