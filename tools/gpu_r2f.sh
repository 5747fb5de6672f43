#!/bin/bash
# (1) TMA-only piece-pattern probe: K1's H -> H' piece map moved by bulk TMA
#     (no shear, no consumer warps) against a plain piece copy and memcpy;
# (2) the autotuner with the task-consumer candidates: C3 / C5 / C2 / C4 bench
#     lines (kernel only) with LFBP_TUNE_LOG.
mkdir -p gpurun_out; o=gpurun_out/r2f.jsonl; : > $o
P=tools/tma_pattern_probe
for st in 2 3 4; do timeout 120 $P 631 21 21 2528 16 0 0 $st 20 >> $o 2>&1; done
timeout 120 $P 631 21 21 2528 16 0 1 3 20 >> $o 2>&1
timeout 120 $P 631 21 21 2528 16 1 0 3 20 >> $o 2>&1
timeout 120 $P 631 21 21 2528 16 2 0 3 20 >> $o 2>&1
timeout 120 $P 631 21 21 2528 16 0 0 2 20 2 >> $o 2>&1
timeout 120 $P 399 19 19 1600 64 0 0 4 10 >> $o 2>&1
timeout 120 $P 399 19 19 1600 64 2 0 4 10 >> $o 2>&1
timeout 120 $P 195 15 15 784 51 0 0 4 50 >> $o 2>&1
timeout 120 $P 195 15 15 784 51 2 0 4 50 >> $o 2>&1
timeout 120 $P 195 15 15 3136 51 0 0 3 50 >> $o 2>&1
for c in C3 C5 C2 C4; do
  LFBP_TUNE_LOG=1 timeout 900 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/r2f_bench_$c.json 2> gpurun_out/r2f_bench_$c.err
done
true
