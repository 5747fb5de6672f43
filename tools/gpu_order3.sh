#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? | tee -a gpurun_out/pytest_gpu.log
timeout 300 python tools/fuzz_parity.py --cases 200 --seed 23 > gpurun_out/fuzz3.log 2>&1; tail -1 gpurun_out/fuzz3.log
timeout 900 python tools/paper_shapes.py > gpurun_out/paper_shapes.jsonl 2>&1; echo shapes_rc=$?
true
