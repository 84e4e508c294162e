#!/bin/bash
# Batched comparator vs the sample-wise engines at c4 / c5 dims (SURVEY
# §8(f) row 1): reference-schema CSV per mode, batch-size sweep; batched runs
# until it reports oom.
set -u
mkdir -p gpurun_out
C4="--frames 1000 --labels 200 --joint 512 --vocab 1024 --warmup 1 --steps 3"
C5="--frames 750 --labels 150 --joint 640 --vocab 4096 --warmup 1 --steps 3"
for m in batched sample_wise sample_wise_pr_dp; do
  python report.py sweep --mode $m --axis batch --values 8,32,64,96,128 $C4 \
    > gpurun_out/modes_c4_$m.csv 2>gpurun_out/modes_c4_$m.err
  python report.py sweep --mode $m --axis batch --values 8,16,32 $C5 \
    > gpurun_out/modes_c5_$m.csv 2>gpurun_out/modes_c5_$m.err
done
tail -n +1 gpurun_out/modes_c*.csv
