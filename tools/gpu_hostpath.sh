#!/bin/bash
# host paths after the staging-thread default change: first call in a fresh process, drop-in and C-ABI timings
mkdir -p gpurun_out
timeout 300 python tools/first_call.py > gpurun_out/first_call.jsonl 2>&1; echo first_rc=$?
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.jsonl 2>&1; echo e2e_rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 300 -k "host or dropin or multi" > gpurun_out/pytest_host.log 2>&1; echo pytest_rc=$? | tee -a gpurun_out/pytest_host.log
true
