#!/bin/bash
# K1 debug builds (round 2 investigation of C5/C3): no-LDS and no-store consumers
mkdir -p gpurun_out; o=gpurun_out/pattern2.jsonl; : > $o
for lib in new NOLDS NOSTORE new; do
  if [ $lib = new ]; then L=; else L=abtest/libhprime_$lib.so; fi
  LFBP_LIB_PATH=$L timeout 300 python tools/k1_probe.py 631,631,21,21,16 --tag $lib >> $o 2>&1
  LFBP_LIB_PATH=$L timeout 300 python tools/k1_probe.py 399,399,19,19,64 --tag $lib >> $o 2>&1
  LFBP_LIB_PATH=$L timeout 300 python tools/k1_probe.py 195,195,15,15,51 --tag $lib --reps 100 >> $o 2>&1
  LFBP_LIB_PATH=$L timeout 300 python tools/k1_probe.py 273,273,13,13,41 --f64 --tag $lib --reps 100 >> $o 2>&1
done
true
