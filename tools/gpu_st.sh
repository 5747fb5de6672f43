#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/st.jsonl; : > $o
K="LFBP_AUTOTUNE=0 LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 LFBP_KFLAGS=24"
K2="LFBP_AUTOTUNE=0 LFBP_STAGES=3 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=8"
for r in 1 2; do
for lib in base st1 st2 st3; do
  if [ $lib = base ]; then L=; else L=abtest/libhprime_$lib.so; fi
  env $K LFBP_LIB_PATH=$L timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 24 --gap 2 --tag C5_$lib >> $o 2>&1
  sleep 3
  env $K2 LFBP_LIB_PATH=$L timeout 300 python tools/phase_trace.py 195,195,15,15,51 --bursts 1 --launches 800 --gap 2 --tag C2_$lib >> $o 2>&1
  sleep 3
done; done
true
