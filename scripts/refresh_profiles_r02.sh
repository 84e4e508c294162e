# Copy the round-2 final evidence (scripts/gpu_r2_final.sh) from gpurun_out/
# into the committed profiles/ files (summaries regenerated from the raw captures).
set -e
cd "$(dirname "$0")/.."
G=gpurun_out; P=profiles
grep '^{' $G/bench_default.json | tail -n1 > $P/r02_bench_c4_default.json
grep '^{' $G/bench_reference.json | tail -n1 > $P/r02_bench_c4_reference_arm.json
for c in c1 c2 c3 c5 c4_tf32 c4_bf16x; do
  [ -f $G/bench_$c.json ] && grep '^{' $G/bench_$c.json | tail -n1 > $P/r02_bench_$c.json
done
grep '^{' $G/bench_shared2.json | tail -n1 > $P/r02_bench_c3_2rank_shared_gpu.json || true
cp $G/launches_c4.csv $P/r02_ncu_launch_list_c4.csv
python scripts/ncu_shares.py $G/launches_c4.csv > $P/r02_ncu_launch_shares_c4.txt
ncu -i $G/prof_c4.ncu-rep --page raw --csv > /tmp/prof_c4_raw_r02.csv 2>/dev/null
python scripts/ncu_summary.py /tmp/prof_c4_raw_r02.csv > $P/r02_ncu_full_c4_summary.txt
python scripts/ncu_traffic.py /tmp/prof_c4_raw_r02.csv $P/r02_ncu_traffic.json > /dev/null
cp $G/ref_parity.log $P/r02_cpp_ref_parity.jsonl
tail -1 $G/pytest_gpu.log > $P/r02_pytest_gpu_tail.txt
for t in memcheck racecheck synccheck initcheck; do echo "== $t"; grep -E "SUMMARY|^fp16|^bf16" $G/sanitize_$t.log; done > $P/r02_sanitize_summary.txt
cp $G/sanitize_racecheck.log $P/r02_sanitize_racecheck.log
cuobjdump -sass paper_2211_16270_b200/libswt_b200.so | grep -oE "\b(UTCHMMA(\.2CTA)?|UTMALDG\.[0-9A-Z.]+|UTMASTG\.[0-9A-Z.]+|LDTM\.[x0-9]+|HMMA|HGMMA)\b" | sort | uniq -c > $P/r02_sass_census.txt
echo refreshed
