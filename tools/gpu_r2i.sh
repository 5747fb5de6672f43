#!/bin/bash
# C5 headline with the grid-capped candidates in the tuner; ncu --set full of
# K1 on a 16-plane C5 slab with the chosen plan pinned; launch list.
mkdir -p gpurun_out; L=gpurun_out/r2i.log; : > $L
LFBP_TUNE_LOG=1 timeout 1500 python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
echo "bench rc=$?" >> $L
K=$(python -c "import json;print(' '.join(map(str,json.load(open('gpurun_out/r2i_bench.json'))['config']['kernel_plan']['knobs'])))")
set -- $K
echo "knobs $K" >> $L
export LFBP_STAGES=$1 LFBP_STAGE_KB=$2 LFBP_CONSUMER_WARPS=$3 LFBP_SUBWARP=$4 LFBP_KFLAGS=$5 LFBP_GRID=$6
timeout 900 python tools/k1_probe.py 631,631,21,21,16 --tag C5slab_pinned >> $L 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:hprime_kernel -s 1 -c 1 \
  -o gpurun_out/r2i_c5slab python tools/ncu_one.py 631,631,21,21,16 > gpurun_out/r2i_ncu.log 2>&1
echo "ncu rc=$?" >> $L
true
