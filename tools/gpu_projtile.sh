#!/bin/bash
# projector tile shape sweep (rows per thread x coarse columns per block), C2 PSF / 512^2 and C4 / 512^2
mkdir -p gpurun_out
o=gpurun_out/proj_tile_sweep.jsonl; : > $o
for psf in C2 C4; do
for rl in "" 5 7 9 13; do for tk in "" 18 12; do
LFBP_PROJ_RL=$rl LFBP_PROJ_TK=$tk timeout 300 python tools/proj_bench.py --psf $psf --image 512 --quick >> $o 2>&1
done; done; done
true
