#!/bin/bash
# C5-row pattern: stride between a unit's runs (n_t) vs throughput; read-only / write-only variants
mkdir -p gpurun_out; o=gpurun_out/stride.jsonl; : > $o
for sh in 631,631,21,21,16 631,63,21,21,160 631,127,21,21,80 631,317,21,21,32 631,1263,21,21,8 631,631,21,21,16; do
  LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 timeout 300 python tools/k1_probe.py $sh --tag fixed >> $o 2>&1
done
for sh in 399,399,19,19,64 399,41,19,19,620; do
  LFBP_STAGES=2 LFBP_STAGE_KB=96 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=16 timeout 300 python tools/k1_probe.py $sh --tag fixed >> $o 2>&1
done
for lib in WONLY NOSTORE NOLDS; do
  LFBP_LIB_PATH=abtest/libhprime_$lib.so LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 timeout 300 python tools/k1_probe.py 631,631,21,21,16 --tag $lib >> $o 2>&1
  LFBP_LIB_PATH=abtest/libhprime_$lib.so LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 timeout 300 python tools/k1_probe.py 631,63,21,21,160 --tag $lib >> $o 2>&1
done
true
