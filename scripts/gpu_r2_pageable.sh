# pageable host buffers through the pinned staging rings: full GPU suite, C++ drop-in parity, bench (pinned + pageable e2e)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 ./oracle/_ref/ref_parity > gpurun_out/ref_parity.log 2>&1; tail -2 gpurun_out/ref_parity.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; python scripts/bench_summary.py gpurun_out/bench_c4.log
python - <<'P'
import json
d=json.loads([l for l in open('gpurun_out/bench_c4.log') if l.startswith('{')][-1])
print(json.dumps(d['e2e']))
P
