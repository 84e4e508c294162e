# bench lines for every BASELINE config and the three precisions at c4
set -x
mkdir -p gpurun_out
for cfg in c1 c2 c3 c5; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$cfg.json 2>&1
  python scripts/bench_summary.py gpurun_out/bench_$cfg.json
done
for p in tf32 bf16x; do
  timeout 900 python bench.py --precision $p --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_$p.json 2>&1
  python scripts/bench_summary.py gpurun_out/bench_c4_$p.json
done
