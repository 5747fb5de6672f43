#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "cphase" > gpurun_out/cp1_tests.log 2>&1
echo "rc=$?" >> gpurun_out/cp1_tests.log
o=gpurun_out/cp1.jsonl; : > $o
K="LFBP_AUTOTUNE=0 LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32"
for f in 24 88 64 0; do
  env $K LFBP_KFLAGS=$f timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 40 --gap 2 --tag C5_f$f >> $o 2>&1; sleep 3
done
for w in 4 6 12; do
  env $K LFBP_CONSUMER_WARPS=$w LFBP_KFLAGS=88 timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 40 --gap 2 --tag C5_f88_w$w >> $o 2>&1; sleep 3
done
K3="LFBP_AUTOTUNE=0 LFBP_STAGES=4 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=8"
for f in 0 64; do
  env $K3 LFBP_KFLAGS=$f timeout 300 python tools/phase_trace.py 399,399,19,19,64 --bursts 1 --launches 200 --gap 2 --tag C3_f$f >> $o 2>&1; sleep 3
done
K2="LFBP_AUTOTUNE=0 LFBP_STAGES=3 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=8"
for f in 0 64; do
  env $K2 LFBP_KFLAGS=$f timeout 300 python tools/phase_trace.py 195,195,15,15,51 --bursts 1 --launches 1500 --gap 2 --tag C2_f$f >> $o 2>&1; sleep 3
done
K4="LFBP_AUTOTUNE=0 LFBP_STAGES=4 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=16"
for f in 0 64; do
  env $K4 LFBP_KFLAGS=$f timeout 300 python tools/phase_trace.py 273,273,13,13,41 --f64 --bursts 1 --launches 600 --gap 2 --tag C4_f$f >> $o 2>&1; sleep 3
done
true
