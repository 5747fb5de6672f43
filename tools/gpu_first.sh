#!/bin/bash
# first call in a fresh process and steady-state calls, pinned (library allocator) vs pageable result array
mkdir -p gpurun_out
o=gpurun_out/first_call.jsonl; : > $o
for m in pinned pageable pinned; do
echo "{\"out_mode\": \"$m\"}" >> $o
LFBP_OUT_MODE=$m timeout 300 python tools/first_call.py --calls 5 >> $o 2>&1
done
timeout 300 python tools/first_call.py --calls 3 --config C4 >> $o 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 300 > gpurun_out/pytest_parity.log 2>&1; echo pytest_rc=$? | tee -a gpurun_out/pytest_parity.log
true
