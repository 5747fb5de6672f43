#!/bin/bash
mkdir -p gpurun_out
timeout 420 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
python tools/stability.py --config C2 --plans "3,48,8,8;3,48,16,16;4,48,8,16" > gpurun_out/stab_c2.jsonl 2>&1
python tools/stability.py --config C3 --plans "4,48,8,16;4,32,16,32;4,48,8,8" --reps 40 > gpurun_out/stab_c3.jsonl 2>&1
python tools/stability.py --config C5 --plans "3,48,8,32;4,48,8,16;3,48,8,16" --reps 10 --rounds 3 > gpurun_out/stab_c5.jsonl 2>&1
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
true
