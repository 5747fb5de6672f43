#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/tlbpf.jsonl; : > $o
K="LFBP_AUTOTUNE=0 LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32"
K3="LFBP_AUTOTUNE=0 LFBP_STAGES=4 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=8"
for r in 1 2; do
  env $K LFBP_KFLAGS=24 timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 24 --gap 2 --tag C5_f24 >> $o 2>&1; sleep 3
  env $K LFBP_KFLAGS=88 timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 24 --gap 2 --tag C5_f88 >> $o 2>&1; sleep 3
  env $K LFBP_KFLAGS=88 LFBP_PF_SHIFT=16 timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 24 --gap 2 --tag C5_f88_64k >> $o 2>&1; sleep 3
  env $K LFBP_KFLAGS=64 timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 24 --gap 2 --tag C5_f64 >> $o 2>&1; sleep 3
  env $K LFBP_KFLAGS=0 timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 24 --gap 2 --tag C5_f0 >> $o 2>&1; sleep 3
  env $K3 LFBP_KFLAGS=0 timeout 300 python tools/phase_trace.py 399,399,19,19,64 --bursts 1 --launches 120 --gap 2 --tag C3_f0 >> $o 2>&1; sleep 3
  env $K3 LFBP_KFLAGS=64 timeout 300 python tools/phase_trace.py 399,399,19,19,64 --bursts 1 --launches 120 --gap 2 --tag C3_f64 >> $o 2>&1; sleep 3
done
true
