#!/bin/bash
# fuzz with the kernel-option knob sets; FP64 DFMA vs DMMA throughput probe
mkdir -p gpurun_out; L=gpurun_out/r2za.log; : > $L
timeout 1800 python tools/fuzz_parity.py --cases 1500 --seed 2029 > gpurun_out/r2za_fuzz.log 2>&1
echo "fuzz rc=$?" >> $L; tail -1 gpurun_out/r2za_fuzz.log >> $L
timeout 300 tools/fp64_peak > gpurun_out/r2za_fp64.jsonl 2>&1
echo "fp64 rc=$?" >> $L
true
