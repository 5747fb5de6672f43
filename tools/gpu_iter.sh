#!/bin/bash
# one optimisation iteration: tests, sweep, bench, ncu of C2 at the default plan
mkdir -p gpurun_out
timeout 420 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 1200 python tools/sweep.py --configs ${SWEEP_CONFIGS:-C2,C4,C3} --grid "${SWEEP_GRID:-STAGES=2,3,4;STAGE_KB=12,16,24,32,48;CONSUMER_WARPS=4,6,8,12}" > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo sweep_rc=$?
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
CMD="python bench.py --config C2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-verify"
$CMD > gpurun_out/plain_c2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hprime_kernel -s 3 -c 1 -o gpurun_out/prof_c2 -f $CMD > gpurun_out/ncu_c2.log 2>&1; echo ncu_rc=$?
[ -n "$E2E_PROBE" ] && { timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.jsonl 2>&1; echo e2e_rc=$?; }
