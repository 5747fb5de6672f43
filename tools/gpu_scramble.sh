#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/scramble.jsonl; : > $o
timeout 300 python tools/order_check.py 631,631,21,21,3 >> $o 2>&1
timeout 300 python tools/order_check.py 40,30,7,5,3 >> $o 2>&1
K="LFBP_AUTOTUNE=0 LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32"
for sh in 631,631,21,21,101 640,631,21,21,99; do
  for f in 16 32 48 24 0; do
    env $K LFBP_KFLAGS=$f timeout 300 python tools/phase_trace.py $sh --bursts 1 --launches 30 --gap 3 --tag f${f}_$sh >> $o 2>&1
    sleep 4
  done
done
true
