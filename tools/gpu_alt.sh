#!/bin/bash
# two plans alternated in one process with NVML state per window
mkdir -p gpurun_out
o=gpurun_out/alternate.jsonl; : > $o
timeout 300 python tools/alternate.py --config C2 --plans "4,48,8,8;2,96,8,8" --cycles 10 --reps 40 >> $o 2>&1
true
