#!/bin/bash
# final-state check: GPU suite, smoke, default bench, reference arm
mkdir -p gpurun_out; L=gpurun_out/r2x.log; : > $L
S=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2x_pytest.log 2>&1
echo "pytest rc=$? secs=$(( $(date +%s) - S ))" >> $L; tail -1 gpurun_out/r2x_pytest.log >> $L
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1
echo "smoke rc=$?" >> $L
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2x_ref.json 2> gpurun_out/r2x_ref.err
echo "ref rc=$?" >> $L
LFBP_TUNE_LOG=1 timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err
echo "bench rc=$?" >> $L
true
