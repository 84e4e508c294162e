# round-2 final evidence: parity suites, C++ drop-in parity, bench (both arms, configs,
# precisions, 2-rank orchestration), ncu launch list + full capture, compute-sanitizer
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 ./oracle/_ref/ref_parity > gpurun_out/ref_parity.log 2>&1; tail -1 gpurun_out/ref_parity.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; python scripts/bench_summary.py gpurun_out/bench_default.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2>&1; tail -c 300 gpurun_out/bench_reference.json
for c in c1 c2 c3 c5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline > gpurun_out/bench_$c.json 2>&1
  python scripts/bench_summary.py gpurun_out/bench_$c.json | head -2
done
for p in tf32 bf16x; do
  timeout 600 python bench.py --precision $p --steps 3 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline > gpurun_out/bench_c4_$p.json 2>&1
  python scripts/bench_summary.py gpurun_out/bench_c4_$p.json | head -2
done
SWTB_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --config c3 > gpurun_out/bench_shared2.json 2>gpurun_out/bench_shared2.err; tail -c 400 gpurun_out/bench_shared2.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
  --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary \
  > gpurun_out/ncu_launch_bench.log 2>&1; tail -1 gpurun_out/ncu_launch_bench.log | cut -c1-200
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
  -k regex:'gemm_kernel|lattice|zslab|zmean|edge|reduce_partials' -c 24 \
  -o gpurun_out/prof_c4 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary \
  > gpurun_out/ncu_full_c4.log 2>&1; tail -1 gpurun_out/ncu_full_c4.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_case.py fp16,bf16 > gpurun_out/sanitize_$t.log 2>&1
  tail -1 gpurun_out/sanitize_$t.log
done
ls -la gpurun_out
