# ncu full capture of the f^O forward and dh GEMMs with and without the
# A-resident mode (c3 step)
mkdir -p gpurun_out
for a in 0 1; do
  SWTB_ARES=$a timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:'EpiFwdLse|EpiBwdDh' \
    -s 8 -c 2 -o gpurun_out/prof_ares$a python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/ncu_ares$a.log 2>&1
done
ls -la gpurun_out/prof_ares*
