#!/bin/bash
# placement sensitivity of K1 plans: H' (then H) at whole-2 MB-page and sub-page offsets
mkdir -p gpurun_out
o=gpurun_out/placement.jsonl; : > $o
P="4,48,8,8;2,96,8,8;4,48,16,16"
timeout 600 python tools/placement.py --config C2 --which dst --offsets 0,1048576,2097152,3145728,5242880,7340032 --plans "$P" >> $o 2>&1
timeout 600 python tools/placement.py --config C2 --which src --offsets 1048576,2097152,3145728,5242880 --plans "$P" >> $o 2>&1
true
