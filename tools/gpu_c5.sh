#!/bin/bash
# smoke + the opt-in full-size C5 parity test (71 GB in + 71 GB out on one GPU)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
LFBP_TEST_C5=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "C5" --timeout 1400 -rs > gpurun_out/pytest_c5.log 2>&1; echo c5_rc=$?
timeout 600 python bench.py --config C5 --steps 20 --no-cpu --no-e2e > gpurun_out/bench_C5.log 2>&1; echo bench_c5_rc=$?
true
