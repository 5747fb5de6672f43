#!/bin/bash
# tests, then the plan sweep, then the bench
mkdir -p gpurun_out
timeout 420 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 1200 python tools/sweep.py --configs C2,C4,C3 --grid "${SWEEP_GRID:-STAGES=2,3,4;STAGE_KB=12,16,24,32;CONSUMER_WARPS=4,6,8;KFLAGS=0,1,2,3}" > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo sweep_rc=$?
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.jsonl 2>&1; echo e2e_rc=$?
