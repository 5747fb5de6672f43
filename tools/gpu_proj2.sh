#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_projector.py -x -q --timeout 250 > gpurun_out/pytest_proj.log 2>&1; echo pytest_rc=$? | tee -a gpurun_out/pytest_proj.log
: > gpurun_out/proj_rl.json
for rl in 0 8; do
LFBP_PROJ_RL=$rl timeout 600 python tools/proj_bench.py --psf C4 --image 512 --iters 2 >> gpurun_out/proj_rl.json 2>&1
LFBP_PROJ_RL=$rl timeout 900 python tools/proj_bench.py --psf C3 --image 512 --iters 1 >> gpurun_out/proj_rl.json 2>&1
done
true
