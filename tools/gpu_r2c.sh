#!/bin/bash
# round-2 evidence pass: GPU suite (C5 included), smoke, C5 headline bench,
# reference arm, ncu launch list of the bench
mkdir -p gpurun_out
L=gpurun_out/r2c.log
S=$(date +%s)
nvidia-smi --query-gpu=name,memory.total,power.limit,clocks.max.sm --format=csv > $L 2>&1
free -g >> $L; nproc >> $L
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2c_pytest.log 2>&1
echo "pytest rc=$? secs=$(( $(date +%s) - S ))" >> $L
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1
echo "smoke rc=$?" >> $L
S=$(date +%s)
timeout 1500 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
echo "bench rc=$? secs=$(( $(date +%s) - S ))" >> $L
S=$(date +%s)
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2c_ref.json 2> gpurun_out/r2c_ref.err
echo "ref rc=$? secs=$(( $(date +%s) - S ))" >> $L
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2c_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/r2c_ncu.log 2>&1
echo "ncu rc=$?" >> $L
true
