#!/bin/bash
# self-resetting ticket slots: checked-build fuzz, full GPU suite, smoke,
# default bench, paper shapes (small launches now tune tickets too)
mkdir -p gpurun_out; L=gpurun_out/r2t.log; : > $L
LFBP_LIB_PATH=abtest/libhprime_CHECKED.so LFBP_KFLAGS=128 timeout 900 python tools/fuzz_parity.py --cases 200 --seed 91 > gpurun_out/r2t_fuzz_checked.log 2>&1
echo "checked fuzz rc=$?" >> $L; tail -1 gpurun_out/r2t_fuzz_checked.log >> $L
S=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2t_pytest.log 2>&1
echo "pytest rc=$? secs=$(( $(date +%s) - S ))" >> $L; tail -1 gpurun_out/r2t_pytest.log >> $L
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1
echo "smoke rc=$?" >> $L
LFBP_TUNE_LOG=1 timeout 1500 python bench.py > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
echo "bench rc=$?" >> $L
timeout 1200 python tools/paper_shapes.py > gpurun_out/r2t_paper_shapes.jsonl 2>&1
echo "paper rc=$?" >> $L
true
