#!/bin/bash
# drop-in host path on a pageable array: memcpy threads x chunk size
mkdir -p gpurun_out
o=gpurun_out/dropin_sweep.jsonl; : > $o
nproc >> $o
for th in 4 8 12 16; do for mb in 34 68 136; do
LFBP_COPY_THREADS=$th LFBP_CHUNK_MB=$mb timeout 300 python tools/e2e_probe.py --dropin-only --modes stage >> $o 2>&1
done; done
timeout 300 python tools/e2e_probe.py >> $o 2>&1
true
