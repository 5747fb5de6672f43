#!/bin/bash
# Working-set (TLB reach) sweep in short windows, then K1 vs copy_ under
# sustained (2 s) load with NVML power / clock sampling.
mkdir -p gpurun_out
o=gpurun_out/r01_power_tlb.jsonl; : > $o
timeout 300 python tools/tlb_probe.py --base 195,195,15 --ny 15,29,45,59,75,91,121 --plan 3,48,8,8 >> $o 2>&1
timeout 300 python tools/tlb_probe.py --base 399,399,19 --ny 3,5,7,9,11,13,15,19,25 --plan 4,48,12,16 >> $o 2>&1
timeout 300 python tools/tlb_probe.py --base 273,273,13 --f64 --ny 7,13,21,27,35,41 --plan 4,48,8,16 >> $o 2>&1
timeout 300 python tools/tlb_probe.py --base 195,195,15 --ny 15 --plan 3,48,8,8 --secs 2 >> $o 2>&1
timeout 300 python tools/tlb_probe.py --base 399,399,19 --ny 19 --plan 4,48,12,16 --secs 2 --gb 29.4 >> $o 2>&1
timeout 300 python tools/tlb_probe.py --base 273,273,13 --f64 --ny 13 --plan 4,48,8,16 --secs 2 >> $o 2>&1
timeout 400 python tools/tlb_probe.py --base 631,631,21 --ny 21 --plan 3,64,8,32 --secs 2 --gb 141.9 >> $o 2>&1
true
