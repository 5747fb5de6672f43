#!/bin/bash
mkdir -p gpurun_out
for f in 0 4; do
  LFBP_KFLAGS=$f python tools/stability.py --config C2 --plans "3,48,8,8;4,48,16,16" --rounds 3 > gpurun_out/order_c2_$f.jsonl 2>&1
  LFBP_KFLAGS=$f python tools/stability.py --config C3 --plans "4,48,12,16;4,48,8,8" --reps 40 --rounds 3 > gpurun_out/order_c3_$f.jsonl 2>&1
  LFBP_KFLAGS=$f python tools/stability.py --config C5 --plans "3,48,8,32;4,48,8,16" --reps 10 --rounds 2 > gpurun_out/order_c5_$f.jsonl 2>&1
  LFBP_KFLAGS=$f python tools/stability.py --config C4 --plans "4,48,8,16;4,32,12,32" --reps 50 --rounds 3 > gpurun_out/order_c4_$f.jsonl 2>&1
done
true
