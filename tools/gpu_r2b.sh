#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do
LFBP_TUNE_LOG=1 timeout 1200 python bench.py --no-cpu --no-e2e > gpurun_out/r2b_bench_$i.json 2> gpurun_out/r2b_bench_$i.err
sleep 5
done
LFBP_TUNE_LOG=1 timeout 1200 python bench.py --config C3 --no-cpu --no-e2e > gpurun_out/r2b_bench_c3.json 2> gpurun_out/r2b_bench_c3.err
true
