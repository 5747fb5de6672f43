#!/bin/bash
# same-box A/B of library builds in abtest/, pinned plans
mkdir -p gpurun_out
o=gpurun_out/ab_lib.jsonl; : > $o
for r in 1 2; do
for lib in ${LIBS:-old new}; do
  if [ $lib = new ]; then L=; else L=abtest/libhprime_$lib.so; fi
  echo "{\"lib\": \"$lib\", \"round\": $r}" >> $o
  LFBP_LIB_PATH=$L timeout 300 python tools/stability.py --config C5 --plans "3,64,8,32" --rounds 2 --reps 40 >> $o 2>&1
  LFBP_LIB_PATH=$L timeout 300 python tools/stability.py --config C3 --plans "2,96,8,16" --rounds 2 --reps 100 >> $o 2>&1
done; done
true
