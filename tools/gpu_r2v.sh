#!/bin/bash
# Evidence for the shipped C5 plan: ncu --set full of K1 on a 16-plane C5 slab
# with the tuned plan pinned (knobs from argv or the r2t bench), and the
# launch list of the default bench.
mkdir -p gpurun_out; L=gpurun_out/r2v.log; : > $L
K=${1:-"4 48 12 8 128 0"}
set -- $K
export LFBP_STAGES=$1 LFBP_STAGE_KB=$2 LFBP_CONSUMER_WARPS=$3 LFBP_SUBWARP=$4 LFBP_KFLAGS=$5 LFBP_GRID=$6
echo "knobs $K" >> $L
timeout 600 python tools/k1_probe.py 631,631,21,21,16 --tag C5slab_pinned >> $L 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:hprime_kernel -s 1 -c 1 \
  -o gpurun_out/r2v_c5slab python tools/ncu_one.py 631,631,21,21,16 > gpurun_out/r2v_ncu.log 2>&1
echo "ncu rc=$?" >> $L
unset LFBP_STAGES LFBP_STAGE_KB LFBP_CONSUMER_WARPS LFBP_SUBWARP LFBP_KFLAGS LFBP_GRID
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2v_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/r2v_launch_ncu.log 2>&1
echo "launches rc=$?" >> $L
true
