# Copy a gpu_evidence.sh / gpu_configs.sh run from gpurun_out/ into the
# committed profiles/ files (summaries regenerated from the raw captures).
set -e
cd "$(dirname "$0")/.."
tail -n1 gpurun_out/bench_default.json > profiles/r01_bench_c4_default.json
tail -n1 gpurun_out/bench_reference.json > profiles/r01_bench_c4_reference_arm.json
cp gpurun_out/launches_c4.csv profiles/r01_ncu_launch_list_c4.csv
python scripts/ncu_shares.py gpurun_out/launches_c4.csv > profiles/r01_ncu_launch_shares_c4.txt
ncu -i gpurun_out/prof_c4.ncu-rep --page raw --csv > /tmp/prof_c4_raw.csv 2>/dev/null
python scripts/ncu_summary.py /tmp/prof_c4_raw.csv > profiles/r01_ncu_full_c4_summary.txt
python scripts/ncu_traffic.py /tmp/prof_c4_raw.csv profiles/r01_ncu_traffic.json > /dev/null
cp gpurun_out/ref_parity.log profiles/r01_cpp_ref_parity.jsonl
tail -1 gpurun_out/pytest_gpu.log > profiles/r01_pytest_gpu_tail.txt
if [ -f gpurun_out/configs.txt ]; then
  cp gpurun_out/configs.txt profiles/r01_bench_configs.txt
  for c in c1 c2 c3 c5 c4_tf32 c4_bf16x; do
    [ -f gpurun_out/bench_$c.json ] && grep '^{' gpurun_out/bench_$c.json | tail -n1 > profiles/r01_bench_$c.json
  done
fi
cuobjdump -sass paper_2211_16270_b200/libswt_b200.so | grep -oE "\b(UTCHMMA(\.2CTA)?|UTMALDG\.[0-9A-Z.]+|UTMASTG\.[0-9A-Z.]+|LDTM\.[x0-9]+|HMMA|HGMMA)\b" | sort | uniq -c > profiles/r01_sass_census.txt
echo refreshed
