#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/proj_rl.json
timeout 600 python tools/proj_bench.py --psf C2 --image 512 --iters 2 >> gpurun_out/proj_rl.json 2>&1
timeout 600 python tools/proj_bench.py --psf C1 --image 256 --iters 2 >> gpurun_out/proj_rl.json 2>&1
true
