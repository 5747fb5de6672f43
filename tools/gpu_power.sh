#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/power.jsonl; : > $o
nvidia-smi -q -d POWER | grep -i "limit" >> gpurun_out/power_limits.txt
for op in copy k1; do
  timeout 120 python tools/power_trace.py 631,631,21,21,24 --secs 4 --op $op >> $o 2>&1
  sleep 5
done
LFBP_LIB_PATH=abtest/libhprime_NOLDS.so timeout 120 python tools/power_trace.py 631,631,21,21,24 --secs 4 --tag nolds >> $o 2>&1
sleep 5
timeout 120 python tools/power_trace.py 399,399,19,19,64 --secs 4 --op k1 >> $o 2>&1
sleep 5
timeout 120 python tools/power_trace.py 195,195,15,15,51 --secs 4 --op k1 >> $o 2>&1
true
