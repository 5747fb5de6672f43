#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/c2_ab.txt; : > $o
for i in 1 2 3; do
  timeout 300 python bench.py --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('auto', d['value'], d['config']['kernel_plan']['knobs'])" >> $o
  LFBP_STAGES=3 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=8 timeout 300 python bench.py --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('3-48-8-8', d['value'])" >> $o
  LFBP_STAGES=2 LFBP_STAGE_KB=96 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=8 timeout 300 python bench.py --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('2-96-8-8', d['value'])" >> $o
  LFBP_STAGES=4 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=16 timeout 300 python bench.py --config C4 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C4 4-48-8-16', d['value'])" >> $o
done
true
