#!/bin/bash
# C5 with tickets: grid caps, diagonal order, consumer shapes (whole array)
mkdir -p gpurun_out; o=gpurun_out/r2u.jsonl; : > $o
run() { tag=$1; shift; env "$@" timeout 300 python tools/k1_probe.py 631,631,21,21,101 --reps 10 --tag $tag >> $o 2>&1; }
for rep in 1 2; do
  for g in 148 146 144 140; do
    run a_g$g LFBP_STAGES=4 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=12 LFBP_SUBWARP=8 LFBP_KFLAGS=128 LFBP_GRID=$g
    run adiag_g$g LFBP_STAGES=4 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=12 LFBP_SUBWARP=8 LFBP_KFLAGS=136 LFBP_GRID=$g
  done
  for w in 8 12 16; do for sw in 8 16; do for st in 3 4; do
    run c_s${st}_w${w}_sw$sw LFBP_STAGES=$st LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=$w LFBP_SUBWARP=$sw LFBP_KFLAGS=128
  done; done; done
  run t_160 LFBP_STAGES=2 LFBP_STAGE_KB=96 LFBP_CONSUMER_WARPS=12 LFBP_KFLAGS=160
  run t_160_w8 LFBP_STAGES=3 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=8 LFBP_KFLAGS=160
done
true
