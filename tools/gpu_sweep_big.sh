#!/bin/bash
# Larger staged units (wider t-bands J) per config.
mkdir -p gpurun_out
o=gpurun_out/r01_sweep_bigstage.jsonl; : > $o
timeout 600 python tools/sweep.py --configs C3,C2 --grid "STAGES=2,3,4;STAGE_KB=48,64,72,96;CONSUMER_WARPS=8,12,16;SUBWARP=8,16,32" >> $o 2>&1
timeout 600 python tools/sweep.py --configs C5 --grid "STAGES=2,3;STAGE_KB=64,112;STAGE_MAX_KB=100,112;CONSUMER_WARPS=8,12,16;SUBWARP=16,32" >> $o 2>&1
true
