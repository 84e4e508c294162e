# ncu --set full of one launch of each output-layer GEMM (c3 step, after warm-up)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:'EpiFwdLse|EpiBwdDh|EpiDzGate|EpiAtomicDb' -s 12 -c 4 -o gpurun_out/prof_gemm -f \
  python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1
ls -la gpurun_out/prof_gemm.ncu-rep
