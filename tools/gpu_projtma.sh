#!/bin/bash
# TMA double-buffered projector windows: projector tests, then timings with (1) and without (0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_projector.py -x -q -m gpu --timeout 600 > gpurun_out/pytest_proj.log 2>&1; echo proj_rc=$? | tee -a gpurun_out/pytest_proj.log
o=gpurun_out/proj_tma.jsonl; : > $o
for r in 1 2; do for t in 0 1; do
for spec in "C2 512" "C4 512" "C1 256"; do set -- $spec
LFBP_PROJ_TMA=$t timeout 300 python tools/proj_bench.py --psf $1 --image $2 --quick | sed "s/^{/{\"tma\": $t, /" >> $o 2>&1
done; done; done
for t in 0 1; do LFBP_PROJ_TMA=$t timeout 300 python tools/proj_bench.py --psf C3 --image 512 --quick | sed "s/^{/{\"tma\": $t, /" >> $o 2>&1; done
true
