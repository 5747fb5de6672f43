#!/bin/bash
# multiple producer warps: parity, then paper shapes with n_x > 32 (and C2 as control), 1 vs auto producers
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 600 > gpurun_out/pytest_parity.log 2>&1; echo parity_rc=$? | tee -a gpurun_out/pytest_parity.log
timeout 300 python tools/fuzz_parity.py --cases 300 --seed 11 > gpurun_out/fuzz2.log 2>&1; tail -1 gpurun_out/fuzz2.log
o=gpurun_out/producers_ab.jsonl; : > $o
for r in 1 2; do
LFBP_PRODUCERS=1 timeout 600 python tools/paper_shapes.py --only 9,10 --tag p1 >> $o 2>&1
timeout 600 python tools/paper_shapes.py --only 9,10 --tag auto >> $o 2>&1
LFBP_PRODUCERS=3 timeout 600 python tools/paper_shapes.py --only 9 --tag p3 >> $o 2>&1
done
true
