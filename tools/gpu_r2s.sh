#!/bin/bash
# Multi-producer dynamic tickets: parity (unit-order tests), then the wide
# paper shapes (n_x > 32) under the tuner and with forced plans.
mkdir -p gpurun_out; L=gpurun_out/r2s.log; : > $L
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "unit_orders or wide or full_scale" > gpurun_out/r2s_pytest.log 2>&1
echo "pytest rc=$?" >> $L; tail -1 gpurun_out/r2s_pytest.log >> $L
LFBP_KFLAGS=128 LFBP_PRODUCERS=3 timeout 900 python tools/fuzz_parity.py --cases 150 --seed 77 > gpurun_out/r2s_fuzz.log 2>&1
echo "fuzz rc=$?" >> $L; tail -1 gpurun_out/r2s_fuzz.log >> $L
timeout 900 python tools/paper_shapes.py --only 7,8,9,10 > gpurun_out/r2s_paper_wide.jsonl 2>&1
echo "paper wide rc=$?" >> $L
timeout 1200 python tools/sweep.py --configs 181x181x95x55x11,307x307x51x51x11 --grid "STAGES=2,3,4;STAGE_KB=32,48,64,96;CONSUMER_WARPS=8,12,16;SUBWARP=4,8,16;KFLAGS=128" > gpurun_out/r2s_sweep_wide.jsonl 2>&1
echo "sweep rc=$?" >> $L
true
