#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_projector.py -x -q --timeout 250 > gpurun_out/pytest_proj.log 2>&1; echo pytest_rc=$? | tee -a gpurun_out/pytest_proj.log
timeout 600 python tools/proj_bench.py --psf C2 --image 512 --iters 2 > gpurun_out/proj_c2.json 2>&1
true
