#!/bin/bash
# producer warps 1 / 2 / 3 on the BASELINE configs and the wide Table 1 shapes (pinned plans)
mkdir -p gpurun_out
o=gpurun_out/ab_prod.jsonl; : > $o
for pr in 1 2 3; do
  echo "{\"producers\": $pr}" >> $o
  LFBP_PRODUCERS=$pr timeout 300 python tools/stability.py --config C5 --plans "3,64,8,32" --rounds 2 --reps 40 >> $o 2>&1
  LFBP_PRODUCERS=$pr timeout 300 python tools/stability.py --config C3 --plans "2,96,8,16" --rounds 2 --reps 100 >> $o 2>&1
  LFBP_PRODUCERS=$pr timeout 300 python tools/stability.py --config C4 --plans "4,48,8,16" --rounds 2 --reps 100 >> $o 2>&1
  LFBP_PRODUCERS=$pr timeout 300 python tools/stability.py --config C2 --plans "2,96,8,8;4,48,8,8" --rounds 2 --reps 200 >> $o 2>&1
done
timeout 300 python tools/order_probe.py 181,181,95,55,11 --tiles 55,4 --plan 2,96,8,8 >> $o 2>&1
timeout 300 python tools/order_probe.py 307,307,51,51,11 --tiles 51,4 --plan 2,96,8,8 >> $o 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "plan_variants or wide_shape or full_scale or randomised" > gpurun_out/pytest_ab.log 2>&1; echo pytest_rc=$? | tee -a gpurun_out/pytest_ab.log
true
