#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/order2.jsonl; : > $o
timeout 300 python tools/order_check.py 631,631,21,21,3 >> $o 2>&1
timeout 300 python tools/order_check.py 195,195,15,15,7 >> $o 2>&1
timeout 300 python tools/order_check.py 40,30,7,5,3 >> $o 2>&1
K5="LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32"
for d in 1 2 3 4 7 21; do
  env $K5 LFBP_KFLAGS=8 LFBP_TILE_Y=$d timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 2 --launches 40 --gap 4 --tag C5_diag$d >> $o 2>&1
  sleep 3
done
K3="LFBP_STAGES=2 LFBP_STAGE_KB=96 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=16"
for d in 2 4 19; do
  env $K3 LFBP_KFLAGS=8 LFBP_TILE_Y=$d timeout 300 python tools/phase_trace.py 399,399,19,19,64 --bursts 2 --launches 200 --gap 4 --tag C3_diag$d >> $o 2>&1
  sleep 3
done
true
