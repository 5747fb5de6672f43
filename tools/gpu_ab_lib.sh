#!/bin/bash
# same-box A/B of library builds in abtest/ (LIBS names; "new" = the in-tree build), pinned plans
mkdir -p gpurun_out
o=gpurun_out/ab_lib.jsonl; : > $o
for r in 1 2; do
for lib in ${LIBS:-base new}; do
  if [ $lib = new ]; then L=; else L=abtest/libhprime_$lib.so; fi
  echo "{\"lib\": \"$lib\", \"round\": $r}" >> $o
  LFBP_LIB_PATH=$L timeout 300 python tools/stability.py --config C5 --plans "3,64,8,32" --rounds 2 --reps 40 >> $o 2>&1
  LFBP_LIB_PATH=$L timeout 300 python tools/stability.py --config C3 --plans "2,96,8,16" --rounds 2 --reps 100 >> $o 2>&1
  LFBP_LIB_PATH=$L timeout 300 python tools/stability.py --config C4 --plans "4,48,8,16" --rounds 2 --reps 100 >> $o 2>&1
  LFBP_LIB_PATH=$L timeout 300 python tools/stability.py --config C2 --plans "2,96,8,8;4,48,8,8" --rounds 2 --reps 200 >> $o 2>&1
done; done
true
