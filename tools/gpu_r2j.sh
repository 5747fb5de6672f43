#!/bin/bash
# Grid cap on the FULL C5 array (142 GB) vs the 16-plane slab, same box.
mkdir -p gpurun_out; o=gpurun_out/r2j.jsonl; : > $o
K="LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 LFBP_KFLAGS=8"
for rep in 1 2; do
for g in 148 146 145 144 142 140 138 136 132 128; do
  env $K LFBP_GRID=$g timeout 300 python tools/k1_probe.py 631,631,21,21,101 --reps 10 --tag full_g$g >> $o 2>&1
done
for g in 145 144 140; do
  env $K LFBP_GRID=$g timeout 300 python tools/k1_probe.py 631,631,21,21,16 --tag slab_g$g >> $o 2>&1
  env $K LFBP_GRID=$g timeout 300 python tools/k1_probe.py 631,631,21,21,50 --reps 10 --tag half_g$g >> $o 2>&1
done
done
true
