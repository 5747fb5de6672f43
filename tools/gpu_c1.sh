#!/bin/bash
# C1 (26 MB, latency-bound) plan probe through bench.py (L2 flushed between steps)
mkdir -p gpurun_out
o=gpurun_out/c1_plans.txt; : > $o
run() { echo "== $*" >> $o; env "$@" timeout 120 python bench.py --config C1 --steps 200 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['config']['kernel_plan']; print(d['roofline']['kernel_ms_avg'], d['value'], k['J'], k['stages'], k['threads'], k['ctas_per_sm'], k['grid'], k['n_units'], k['sub_width'])" >> $o; }
run LFBP_X=0
for W in 2 4; do for cw in 4 6 8; do for st in 2 4; do
run LFBP_SUBWARP=$W LFBP_CONSUMER_WARPS=$cw LFBP_STAGE_KB=8 LFBP_STAGES=$st
done; done; done
run LFBP_SUBWARP=4 LFBP_CONSUMER_WARPS=8 LFBP_STAGE_KB=4 LFBP_STAGES=4
run LFBP_SUBWARP=4 LFBP_CONSUMER_WARPS=8 LFBP_BAND=1 LFBP_STAGES=4
true
