#!/bin/bash
# pruned candidate list: GPU suite, smoke, default bench, reference arm,
# C2-C4 lines, paper shapes
mkdir -p gpurun_out; L=gpurun_out/r2w.log; : > $L
S=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2w_pytest.log 2>&1
echo "pytest rc=$? secs=$(( $(date +%s) - S ))" >> $L; tail -1 gpurun_out/r2w_pytest.log >> $L
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1
echo "smoke rc=$?" >> $L
S=$(date +%s)
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2w_ref.json 2> gpurun_out/r2w_ref.err
echo "ref rc=$? secs=$(( $(date +%s) - S ))" >> $L
S=$(date +%s)
LFBP_TUNE_LOG=1 timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2w_bench.json 2> gpurun_out/r2w_bench.err
echo "bench rc=$? secs=$(( $(date +%s) - S ))" >> $L
for c in C2 C3 C4; do
  LFBP_TUNE_LOG=1 timeout 900 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/r2w_bench_$c.json 2> gpurun_out/r2w_bench_$c.err
  echo "bench $c rc=$?" >> $L
done
timeout 1200 python tools/paper_shapes.py > gpurun_out/r2w_paper_shapes.jsonl 2>&1
echo "paper rc=$?" >> $L
true
