#!/bin/bash
# one long launch vs z-chunked launches on the full C5 array
mkdir -p gpurun_out; o=gpurun_out/r2k.jsonl; : > $o
K="LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 LFBP_KFLAGS=8"
for g in 145 140 148; do
  env $K LFBP_GRID=$g timeout 600 python tools/zchunk_probe.py 631,631,21,21,101 --chunks 0,4,8,16,26,51 --tag g$g >> $o 2>&1
done
env LFBP_STAGES=2 LFBP_STAGE_KB=96 LFBP_CONSUMER_WARPS=12 LFBP_SUBWARP=32 timeout 600 python tools/zchunk_probe.py 399,399,19,19,64 --chunks 0,4,8,16,32 --reps 20 --tag C3 >> $o 2>&1
true
