#!/bin/bash
# Where does K1 lose on the C5 row geometry?  (1) the DRAM piece pattern alone
# (pattern_probe: same pieces, no shear), (2) K1 debug builds without smem
# reads / without stores / without loads, (3) the shipped build.
mkdir -p gpurun_out; o=gpurun_out/r2d.jsonl; : > $o
P=tools/pattern_probe
for lay in 0 1; do
  timeout 120 $P 631 21 21 2528 16 $lay 0 20 >> $o 2>&1
done
timeout 120 $P 195 15 15 784 51 0 0 50 >> $o 2>&1
timeout 120 $P 399 19 19 1600 64 0 0 10 >> $o 2>&1
for lib in new NOLDS NOSTORE NOLOAD new; do
  if [ $lib = new ]; then L=; else L=abtest/libhprime_$lib.so; fi
  LFBP_LIB_PATH=$L timeout 300 python tools/k1_probe.py 631,631,21,21,16 --tag $lib >> $o 2>&1
  LFBP_LIB_PATH=$L timeout 300 python tools/k1_probe.py 195,195,15,15,51 --tag $lib --reps 100 >> $o 2>&1
done
true
