# A/B of engine knobs on the c4 bench (env vars), one line each
set -x
mkdir -p gpurun_out
for cfg in ${AB_CFGS:-"SWTB_PARTS=1" "SWTB_PARTS=2" "SWTB_PARTS=3"}; do
  env $cfg timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$(echo $cfg | tr '= ' '__').log 2>&1
  echo "== $cfg"; python scripts/bench_summary.py gpurun_out/ab_$(echo $cfg | tr '= ' '__').log
done
