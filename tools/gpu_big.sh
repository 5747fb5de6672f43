#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/big_plans.jsonl; : > $o
for pl in 4,16,4,4 4,16,8,4 4,16,16,4 4,16,16,8 4,16,16,16 4,16,8,8 4,16,12,8 2,16,16,8 2,16,16,4; do
timeout 120 python tools/tlb_probe.py --base 181,181,95 --ny 55 --gb 15 --plan $pl --secs 0.3 >> $o 2>&1
done
true
