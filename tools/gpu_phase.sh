#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/phase.jsonl; : > $o
K="LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32"
env $K timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 3 --launches 60 --gap 5 --tag full >> $o 2>&1
sleep 5
env $K LFBP_GRID=128 timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 2 --launches 40 --gap 5 --tag grid128 >> $o 2>&1
sleep 5
env $K LFBP_GRID=100 timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 2 --launches 40 --gap 5 --tag grid100 >> $o 2>&1
sleep 5
env LFBP_STAGES=2 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 2 --launches 40 --gap 5 --tag stages2 >> $o 2>&1
sleep 5
timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 2 --launches 40 --gap 5 --op copy --tag copy >> $o 2>&1
true
