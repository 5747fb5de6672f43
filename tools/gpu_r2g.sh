#!/bin/bash
# Persistent-grid size sweep (LFBP_GRID = SMs given a CTA) on the tuned plans:
# the C5 tuner picked 140 of 148 SMs (+9 %); where is the optimum?
mkdir -p gpurun_out; o=gpurun_out/r2g.jsonl; : > $o
run() { tag=$1; shape=$2; args=$3; shift 3; env "$@" timeout 300 python tools/k1_probe.py $shape $args --tag $tag >> $o 2>&1; }
C5K="LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32"
for rep in 1 2; do
for g in 148 144 140 136 132 128 120 112 96; do
  run C5_f8_g$g 631,631,21,21,16 "" $C5K LFBP_KFLAGS=8 LFBP_GRID=$g
  run C5_f0_g$g 631,631,21,21,16 "" $C5K LFBP_KFLAGS=0 LFBP_GRID=$g
done
for g in 140 128 120; do run C5_f8_s2_g$g 631,631,21,21,16 "" LFBP_STAGES=2 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 LFBP_KFLAGS=8 LFBP_GRID=$g; done
for g in 148 140 132 124 116; do
  run C3_g$g 399,399,19,19,64 "" LFBP_STAGES=2 LFBP_STAGE_KB=96 LFBP_CONSUMER_WARPS=12 LFBP_SUBWARP=32 LFBP_GRID=$g
  run C3_f8_g$g 399,399,19,19,64 "" LFBP_STAGES=2 LFBP_STAGE_KB=96 LFBP_CONSUMER_WARPS=12 LFBP_SUBWARP=32 LFBP_KFLAGS=8 LFBP_GRID=$g
  run C2_T_g$g 195,195,15,15,51 "--reps 100" LFBP_STAGES=2 LFBP_STAGE_KB=96 LFBP_CONSUMER_WARPS=12 LFBP_KFLAGS=32 LFBP_GRID=$g
  run C2_g$g 195,195,15,15,51 "--reps 100" LFBP_STAGES=4 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=12 LFBP_SUBWARP=16 LFBP_GRID=$g
  run C4_g$g 273,273,13,13,41 "--f64 --reps 100" LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 LFBP_KFLAGS=8 LFBP_GRID=$g
done
done
true
