#!/bin/bash
# full GPU suite, benches and the paper shapes
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? | tee -a gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config C1 --steps 200 --no-cpu --no-e2e > gpurun_out/bench_C1.log 2>&1; echo bench_C1_rc=$?
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; echo bench_rc=$?
timeout 300 python bench.py --config C3 --steps 50 --no-cpu --no-e2e > gpurun_out/bench_C3.log 2>&1; echo bench_C3_rc=$?
timeout 600 python tools/paper_shapes.py > gpurun_out/paper_shapes.jsonl 2>&1; echo shapes_rc=$?
true
