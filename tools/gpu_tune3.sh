#!/bin/bash
# autotuner choice stability: three C2 bench processes with the tuner log, then C3-C5, then the GPU suite
mkdir -p gpurun_out
for k in 1 2 3; do
LFBP_TUNE_LOG=1 timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench_tune$k.log 2>&1; echo bench_rc=$?
done
for c in C1 C3 C4 C5; do
LFBP_TUNE_LOG=1 timeout 600 python bench.py --config $c --steps 50 --no-cpu --no-e2e > gpurun_out/bench_$c.log 2>&1; echo bench_${c}_rc=$?
done
timeout 900 python -m pytest tests -x -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? | tee -a gpurun_out/pytest_gpu.log
true
