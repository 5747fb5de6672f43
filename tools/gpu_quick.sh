#!/bin/bash
# full GPU suite, then the C1 bench line
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? | tee -a gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config C1 --steps 200 --no-cpu --no-e2e > gpurun_out/bench_C1.log 2>&1; echo bench_C1_rc=$?
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
true
