#!/bin/bash
# Tuned kernel-only bench lines C1-C5 with the dynamic-ticket candidates;
# the paper's Table 1 geometries against copy_.
mkdir -p gpurun_out; L=gpurun_out/r2r.log; : > $L
for c in C5 C2 C3 C4 C1; do
  LFBP_TUNE_LOG=1 timeout 900 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/r2r_bench_$c.json 2> gpurun_out/r2r_bench_$c.err
  echo "bench $c rc=$?" >> $L
done
timeout 1200 python tools/paper_shapes.py > gpurun_out/r2r_paper_shapes.jsonl 2>&1
echo "paper shapes rc=$?" >> $L
true
