#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_projector.py -x -q --timeout 250 > gpurun_out/pytest_proj.log 2>&1; echo pytest_rc=$? | tee -a gpurun_out/pytest_proj.log
: > gpurun_out/proj_pipe.json
for pp in 1 0; do
LFBP_PROJ_PIPE=$pp timeout 600 python tools/proj_bench.py --psf C2 --image 512 --iters 2 | sed "s/^/pipe=$pp /" >> gpurun_out/proj_pipe.json 2>&1
LFBP_PROJ_PIPE=$pp timeout 600 python tools/proj_bench.py --psf C1 --image 256 --iters 2 | sed "s/^/pipe=$pp /" >> gpurun_out/proj_pipe.json 2>&1
LFBP_PROJ_PIPE=$pp timeout 600 python tools/proj_bench.py --psf C4 --image 512 --iters 1 | sed "s/^/pipe=$pp /" >> gpurun_out/proj_pipe.json 2>&1
done
true
