#!/bin/bash
# Dynamic unit scheduling (HP_FLAG_DYNAMIC = 128): parity, then A/B against
# static interleaving and z-chunked launches on C2-C5 (full arrays).
mkdir -p gpurun_out; L=gpurun_out/r2m.log; : > $L
LFBP_KFLAGS=128 timeout 900 python tools/fuzz_parity.py --cases 200 --seed 13 > gpurun_out/r2m_fuzz.log 2>&1
echo "fuzz128 rc=$?" >> $L; tail -1 gpurun_out/r2m_fuzz.log >> $L
LFBP_KFLAGS=168 timeout 900 python tools/fuzz_parity.py --cases 100 --seed 17 > gpurun_out/r2m_fuzz2.log 2>&1
echo "fuzz168 rc=$?" >> $L; tail -1 gpurun_out/r2m_fuzz2.log >> $L
LFBP_KFLAGS=136 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "baseline_config and not C5" > gpurun_out/r2m_parity.log 2>&1
echo "parity rc=$?" >> $L; tail -1 gpurun_out/r2m_parity.log >> $L
o=gpurun_out/r2m.jsonl; : > $o
run() { tag=$1; shape=$2; args=$3; shift 3; env "$@" timeout 300 python tools/k1_probe.py $shape $args --tag $tag >> $o 2>&1; }
C5K="LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32"
for rep in 1 2; do
  for f in 8 72 136 128 200; do for g in 148 145; do
    run C5_f${f}_g$g 631,631,21,21,101 "--reps 10" $C5K LFBP_KFLAGS=$f LFBP_GRID=$g
  done; done
  for f in 0 128; do run C3_f$f 399,399,19,19,64 "" LFBP_STAGES=2 LFBP_STAGE_KB=96 LFBP_CONSUMER_WARPS=12 LFBP_SUBWARP=32 LFBP_KFLAGS=$f; done
  for f in 32 160; do run C2_f$f 195,195,15,15,51 "--reps 100" LFBP_STAGES=2 LFBP_STAGE_KB=96 LFBP_CONSUMER_WARPS=12 LFBP_KFLAGS=$f; done
  for f in 8 136; do run C4_f$f 273,273,13,13,41 "--f64 --reps 100" LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32 LFBP_KFLAGS=$f; done
done
true
