#!/bin/bash
# C1 (26 MB, latency-bound) plan probe through bench.py (L2 flushed between steps)
mkdir -p gpurun_out
o=gpurun_out/c1_plans.txt; : > $o
run() { echo "== $*" >> $o; env "$@" timeout 120 python bench.py --config C1 --steps 200 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['config']['kernel_plan']; print(d['roofline']['kernel_ms_avg'], d['value'], k['J'], k['stages'], k['threads'], k['ctas_per_sm'], k['grid'], k['n_units'])" >> $o; }
run LFBP_X=0
run LFBP_STAGE_KB=8 LFBP_STAGES=4 LFBP_CONSUMER_WARPS=4
run LFBP_STAGE_KB=8 LFBP_STAGES=2 LFBP_CONSUMER_WARPS=4
run LFBP_STAGE_KB=16 LFBP_STAGES=4 LFBP_CONSUMER_WARPS=8
run LFBP_STAGE_KB=16 LFBP_STAGES=2 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=8
run LFBP_STAGE_KB=4 LFBP_STAGES=2 LFBP_CONSUMER_WARPS=2
run LFBP_STAGE_KB=32 LFBP_STAGES=3 LFBP_CONSUMER_WARPS=12
run LFBP_STAGE_KB=48 LFBP_STAGES=4 LFBP_CONSUMER_WARPS=12 LFBP_CTAS_PER_SM=1
run LFBP_STAGE_KB=8 LFBP_STAGES=3 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=8
true
