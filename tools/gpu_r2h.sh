#!/bin/bash
# Finer persistent-grid sweep around the C5 optimum (144 of 148 SMs), ring
# depth 4 (more bytes in flight per SM), and 144/146 on C2-C4.
mkdir -p gpurun_out; o=gpurun_out/r2h.jsonl; : > $o
run() { tag=$1; shape=$2; args=$3; shift 3; env "$@" timeout 300 python tools/k1_probe.py $shape $args --tag $tag >> $o 2>&1; }
C5K="LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32"
for rep in 1 2; do
for g in 148 147 146 145 144 143 142; do
  run C5_s3_g$g 631,631,21,21,16 "" $C5K LFBP_STAGES=3 LFBP_KFLAGS=8 LFBP_GRID=$g
done
for g in 148 146 144 140 136; do
  run C5_s4_g$g 631,631,21,21,16 "" $C5K LFBP_STAGES=4 LFBP_KFLAGS=8 LFBP_GRID=$g
  run C5_s4w12_g$g 631,631,21,21,16 "" LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=12 LFBP_SUBWARP=32 LFBP_STAGES=4 LFBP_KFLAGS=8 LFBP_GRID=$g
done
for g in 148 146 144; do
  run C3_g$g 399,399,19,19,64 "" LFBP_STAGES=2 LFBP_STAGE_KB=96 LFBP_CONSUMER_WARPS=12 LFBP_SUBWARP=32 LFBP_GRID=$g
  run C3_f8_g$g 399,399,19,19,64 "" LFBP_STAGES=4 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 LFBP_KFLAGS=8 LFBP_GRID=$g
  run C2_T_g$g 195,195,15,15,51 "--reps 100" LFBP_STAGES=2 LFBP_STAGE_KB=96 LFBP_CONSUMER_WARPS=12 LFBP_KFLAGS=32 LFBP_GRID=$g
  run C4_g$g 273,273,13,13,41 "--f64 --reps 100" LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 LFBP_KFLAGS=8 LFBP_GRID=$g
done
done
# full C5 (142 GB) at the candidate optimum, long window with NVML
LFBP_STAGES=3 $C5K LFBP_KFLAGS=8 LFBP_GRID=144 timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 60 --gap 1 --tag C5_g144 > gpurun_out/r2h_phase_g144.json 2>&1
LFBP_STAGES=3 $C5K LFBP_KFLAGS=8 LFBP_GRID=148 timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 60 --gap 1 --tag C5_g148 > gpurun_out/r2h_phase_g148.json 2>&1
true
