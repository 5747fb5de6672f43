#!/bin/bash
# round-end style check: full gpu suite, smoke, default bench, reference arm
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?
true
