#!/bin/bash
# small paper shapes: plan probe (below the autotuner's size)
mkdir -p gpurun_out
o=gpurun_out/small_shapes.jsonl; : > $o
S=0,1,4,5
timeout 200 python tools/paper_shapes.py --only $S --tag default >> $o 2>&1
for band in 1 2 3; do
  LFBP_BAND=$band timeout 200 python tools/paper_shapes.py --only $S --tag band$band >> $o 2>&1
done
LFBP_BAND=2 LFBP_SUBWARP=4 LFBP_CONSUMER_WARPS=4 LFBP_STAGES=4 timeout 200 python tools/paper_shapes.py --only $S --tag band2_w4_cw4 >> $o 2>&1
LFBP_BAND=1 LFBP_SUBWARP=4 LFBP_CONSUMER_WARPS=4 LFBP_STAGES=4 timeout 200 python tools/paper_shapes.py --only $S --tag band1_w4_cw4 >> $o 2>&1
LFBP_BAND=2 LFBP_SUBWARP=8 LFBP_CONSUMER_WARPS=8 LFBP_STAGES=4 timeout 200 python tools/paper_shapes.py --only $S --tag band2_w8_cw8 >> $o 2>&1
true
