#!/bin/bash
mkdir -p gpurun_out
LFBP_AUTOTUNE=0 LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 timeout 600 python tools/placement2.py > gpurun_out/place2.jsonl 2>&1
LFBP_KFLAGS=8 LFBP_AUTOTUNE=0 LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 timeout 600 python tools/placement2.py > gpurun_out/place2_diag.jsonl 2>&1
true
