#!/bin/bash
# z-chunked launches (HP_FLAG_ZCHUNK): parity with tiny chunks forced, then the
# C5 headline with the tuner choosing.
mkdir -p gpurun_out; L=gpurun_out/r2l.log; : > $L
LFBP_KFLAGS=64 LFBP_ZCHUNK_MB=1 timeout 900 python tools/fuzz_parity.py --cases 200 --seed 11 > gpurun_out/r2l_fuzz.log 2>&1
echo "fuzz rc=$?" >> $L; tail -1 gpurun_out/r2l_fuzz.log >> $L
LFBP_KFLAGS=72 LFBP_ZCHUNK_MB=2000 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "baseline_config and not C5" > gpurun_out/r2l_parity.log 2>&1
echo "parity rc=$?" >> $L; tail -1 gpurun_out/r2l_parity.log >> $L
LFBP_TUNE_LOG=1 timeout 1500 python bench.py > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err
echo "bench rc=$?" >> $L
true
