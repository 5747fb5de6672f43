#!/bin/bash
mkdir -p gpurun_out
K="LFBP_AUTOTUNE=0 LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32"
env $K LFBP_KFLAGS=88 timeout 900 ncu --set full --import-source on --clock-control none -k regex:hprime_kernel -s 1 -c 1 -o gpurun_out/cp_c5slab python tools/ncu_one.py 631,631,21,21,8 > gpurun_out/ncu_cp_full.log 2>&1
true
