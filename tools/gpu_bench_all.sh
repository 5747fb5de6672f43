#!/bin/bash
# tests, default bench (C2), per-config kernel benches, ncu of the tuned C2 kernel
mkdir -p gpurun_out
timeout 420 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
for c in C1 C3 C4 C5; do
  timeout 600 python bench.py --config $c --steps 20 --no-cpu --no-e2e > gpurun_out/bench_$c.log 2>&1; echo bench_${c}_rc=$?
done
CMD="python bench.py --config C2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-verify"
$CMD > gpurun_out/plain_c2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hprime_kernel -s 28 -c 1 -o gpurun_out/prof_c2 -f $CMD > gpurun_out/ncu_c2.log 2>&1; echo ncu_rc=$?
true
