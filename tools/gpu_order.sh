#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/order.jsonl; : > $o
K5="LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32"
K3="LFBP_STAGES=2 LFBP_STAGE_KB=96 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=16"
K2="LFBP_STAGES=3 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=8"
for f in 8 0 4; do
  env $K5 LFBP_KFLAGS=$f timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 2 --launches 40 --gap 4 --tag C5_f$f >> $o 2>&1
  sleep 4
done
for f in 8 0; do
  env $K3 LFBP_KFLAGS=$f timeout 300 python tools/phase_trace.py 399,399,19,19,64 --bursts 2 --launches 200 --gap 4 --tag C3_f$f >> $o 2>&1
  sleep 4
  env $K2 LFBP_KFLAGS=$f timeout 300 python tools/phase_trace.py 195,195,15,15,51 --bursts 2 --launches 1500 --gap 4 --tag C2_f$f >> $o 2>&1
  sleep 4
done
true
