#!/bin/bash
# full GPU suite, then the evidence refresh
mkdir -p gpurun_out
timeout 420 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? | tee -a gpurun_out/pytest_gpu.log
bash tools/gpu_profiles.sh
