# the fp16 step tests under non-default engine knobs: 1-SM GEMMs with the
# row-mapped backward, the dense backward, tiny backward sub-slabs
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
for cfg in "SWTB_CTA_GROUP=1" "SWTB_SKIP_ZERO_TILES=0" "SWTB_BWD_SLAB_MB=64" "SWTB_PARTS=1" "SWTB_DETERMINISTIC=0"; do
  env $cfg timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "fp16 or skip or zero_weight or large_logits or host" > gpurun_out/pytest_var.log 2>&1
  echo "$cfg: $(tail -1 gpurun_out/pytest_var.log)"; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_var.log | head -3
done
