#!/bin/bash
# same-box A/B of the headline bench (autotuned, default C2) across library builds in abtest/
mkdir -p gpurun_out
o=gpurun_out/ab_bench.txt; : > $o
for r in 1 2 3; do for lib in ${LIBS:-prev7 new}; do
  if [ $lib = new ]; then L=; else L=abtest/libhprime_$lib.so; fi
  LFBP_LIB_PATH=$L timeout 300 python bench.py --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', d['value'], d['config']['kernel_plan']['knobs'], d['clocks']['sm_mhz'])" >> $o
done; done
