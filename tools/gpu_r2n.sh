#!/bin/bash
# round-end style check: GPU suite, smoke, default bench, reference arm
mkdir -p gpurun_out; L=gpurun_out/r2n.log; : > $L
S=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2n_pytest.log 2>&1
echo "pytest rc=$? secs=$(( $(date +%s) - S ))" >> $L; tail -1 gpurun_out/r2n_pytest.log >> $L
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1
echo "smoke rc=$?" >> $L
S=$(date +%s)
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2n_ref.json 2> gpurun_out/r2n_ref.err
echo "ref rc=$? secs=$(( $(date +%s) - S ))" >> $L
S=$(date +%s)
LFBP_TUNE_LOG=1 timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err
echo "bench rc=$? secs=$(( $(date +%s) - S ))" >> $L
true
