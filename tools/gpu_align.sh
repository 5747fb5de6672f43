#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/align.jsonl; : > $o
K="LFBP_AUTOTUNE=0 LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32"
for sh in 631,631,21,21,101 632,631,21,21,101 640,631,21,21,99 631,632,21,21,101; do
  env $K LFBP_KFLAGS=8 timeout 300 python tools/phase_trace.py $sh --bursts 1 --launches 30 --gap 4 --tag diag_$sh >> $o 2>&1
  sleep 4
  env $K LFBP_KFLAGS=0 timeout 300 python tools/phase_trace.py $sh --bursts 1 --launches 30 --gap 4 --tag yfast_$sh >> $o 2>&1
  sleep 4
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for sh in 632,631,21,21,101 640,631,21,21,99; do
  env $K LFBP_KFLAGS=0 timeout 900 ncu --replay-mode application --clock-control none --metrics $M -k regex:hprime_kernel -s 1 -c 1 --csv python tools/ncu_one.py $sh > gpurun_out/ncu_align_$sh.csv 2>&1
done
true
