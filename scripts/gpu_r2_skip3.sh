# tighter zero-tile bound (occupancy x p_max): full GPU suite, C++ parity, bench, sanitizer on the long case
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head -10
grep -E "fp16 c4 B'=8|fp16 c5 full" gpurun_out/pytest_gpu.log | cut -c1-200
timeout 900 ./oracle/_ref/ref_parity > gpurun_out/ref_parity.log 2>&1; tail -1 gpurun_out/ref_parity.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; python scripts/bench_summary.py gpurun_out/bench_default.json
python - <<'P'
import json
d=json.loads([l for l in open('gpurun_out/bench_default.json') if l.startswith('{')][-1])
print(d['roofline']['active_tile_fraction'], d['secondary'], d['e2e']['value'], d['e2e']['pageable']['value'])
P
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_case.py fp16 > gpurun_out/sanitize_memcheck3.log 2>&1; tail -1 gpurun_out/sanitize_memcheck3.log; grep "300 60" gpurun_out/sanitize_memcheck3.log
