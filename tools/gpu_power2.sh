#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/power2.jsonl; : > $o
timeout 300 python tools/power_trace.py 631,631,21,21,101 --secs 4 --op k1 >> $o 2>&1
sleep 10
timeout 300 python tools/power_trace.py 631,631,21,21,101 --secs 4 --op copy >> $o 2>&1
sleep 10
LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 timeout 300 python tools/power_trace.py 631,631,21,21,16 --secs 4 --op k1 --tag slab16 >> $o 2>&1
sleep 10
LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 timeout 300 python tools/power_trace.py 631,631,21,21,101 --secs 4 --op k1 --tag full_fixed >> $o 2>&1
nvidia-smi -q -d TEMPERATURE,POWER,CLOCK > gpurun_out/smi_q.txt
true
