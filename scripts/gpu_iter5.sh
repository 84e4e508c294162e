# parity suite, c4 bench, racecheck re-check, 2-rank torchrun orchestration on one GPU
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
grep -E "c4 B'=8|c5 full" gpurun_out/pytest_gpu.log | cut -c1-300
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1; tail -c 300 gpurun_out/bench_c4.log
python scripts/bench_summary.py gpurun_out/bench_c4.log
SWTB_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --config c3 > gpurun_out/bench_shared2.log 2>&1; tail -c 800 gpurun_out/bench_shared2.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python scripts/sanitize_case.py fp16 > gpurun_out/sanitize_racecheck.log 2>&1
tail -2 gpurun_out/sanitize_racecheck.log; grep -c "lattice" gpurun_out/sanitize_racecheck.log
