#!/bin/bash
mkdir -p gpurun_out
S=$(date +%s)
timeout 1200 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
echo "bench rc=$? secs=$(( $(date +%s) - S ))" > gpurun_out/r2a_tests.log
free -g >> gpurun_out/r2a_tests.log
timeout 1500 python -m pytest tests/test_reference_suite.py -x -q >> gpurun_out/r2a_tests.log 2>&1
true
