#!/bin/bash
# GPU-box check: gpu tests, bench (ours + reference arm), ncu launch list and one full capture of K1.
mkdir -p gpurun_out
set -x
nproc; free -g | head -2
timeout 420 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-verify"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
ncu --set full --clock-control none --import-source on -k regex:hprime_kernel -s 3 -c 1 -o gpurun_out/prof_c2 -f $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
