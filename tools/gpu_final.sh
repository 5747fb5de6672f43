#!/bin/bash
# final round check: full GPU suite, smoke, reference arm, opt-in full-size C5 parity, evidence refresh
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? | tee -a gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? | tee -a gpurun_out/smoke.log
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?
LFBP_TEST_C5=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "C5" --timeout 1400 -rs > gpurun_out/pytest_c5.log 2>&1; echo c5_rc=$? | tee -a gpurun_out/pytest_c5.log
bash tools/gpu_profiles.sh
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.jsonl 2>&1; echo e2e_rc=$?
true
