#!/bin/bash
# C1 floor probe (K1 vs copy_ vs empty launch, L2 flushed / warm); C5-geometry
# unit order (y-fastest vs band-fastest) and working set; one full ncu
# capture of K1 on a C5-geometry slab (8 planes, plan pinned to C5's best).
mkdir -p gpurun_out
timeout 300 python tools/c1_probe.py > gpurun_out/c1_probe.jsonl 2>&1; echo c1_rc=$?
o=gpurun_out/c5_order.jsonl; : > $o
for kf in 0 4; do
timeout 300 python tools/tlb_probe.py --base 631,631,21 --ny 3,7,21 --gb 12 --plan 3,64,8,32 --kflags $kf --secs 0.5 >> $o 2>&1
done
echo order_rc=$?
export LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32
timeout 300 python tools/one_shape.py 631,631,21,21,8 > gpurun_out/c5slab_plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hprime_kernel -s 2 -c 1 -o gpurun_out/prof_c5slab -f python tools/one_shape.py 631,631,21,21,8 > gpurun_out/ncu_c5slab.log 2>&1; echo ncu_rc=$?
true
