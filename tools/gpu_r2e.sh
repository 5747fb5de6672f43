#!/bin/bash
# Task consumer (HP_FLAG_TASKS = 32): parity under forced flags, then A/B.
mkdir -p gpurun_out; L=gpurun_out/r2e.log; : > $L
LFBP_KFLAGS=32 timeout 900 python tools/fuzz_parity.py --cases 300 --seed 7 > gpurun_out/r2e_fuzz.log 2>&1
echo "fuzz rc=$?" >> $L; tail -2 gpurun_out/r2e_fuzz.log >> $L
LFBP_KFLAGS=32 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "not C5" > gpurun_out/r2e_parity.log 2>&1
echo "parity rc=$?" >> $L; tail -2 gpurun_out/r2e_parity.log >> $L
o=gpurun_out/r2e.jsonl; : > $o
run() { tag=$1; shape=$2; args=$3; shift 3; env "$@" timeout 300 python tools/k1_probe.py $shape $args --tag $tag >> $o 2>&1; }
for rep in 1 2; do
  run C5_auto 631,631,21,21,16 ""
  for w in 8 12 16; do for s in 3 4; do
    run C5_T_s${s}_w$w 631,631,21,21,16 "" LFBP_KFLAGS=32 LFBP_STAGES=$s LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=$w
  done; done
  run C3_auto 399,399,19,19,64 ""
  for kb in 48 96; do for w in 8 12; do
    run C3_T_kb${kb}_w$w 399,399,19,19,64 "" LFBP_KFLAGS=32 LFBP_STAGES=4 LFBP_STAGE_KB=$kb LFBP_CONSUMER_WARPS=$w
  done; done
  run C2_auto 195,195,15,15,51 "--reps 100"
  for kb in 48 96; do for w in 8 12; do
    run C2_T_kb${kb}_w$w 195,195,15,15,51 "--reps 100" LFBP_KFLAGS=32 LFBP_STAGES=4 LFBP_STAGE_KB=$kb LFBP_CONSUMER_WARPS=$w
  done; done
  run C4_auto 273,273,13,13,41 "--f64 --reps 100"
  for kb in 48 96; do for w in 8 12; do
    run C4_T_kb${kb}_w$w 273,273,13,13,41 "--f64 --reps 100" LFBP_KFLAGS=32 LFBP_STAGES=4 LFBP_STAGE_KB=$kb LFBP_CONSUMER_WARPS=$w
  done; done
done
# long windows with NVML: SM clock under the power cap
timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 60 --gap 1 --tag C5_auto > gpurun_out/r2e_phase_auto.json 2>&1
LFBP_KFLAGS=32 LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 60 --gap 1 --tag C5_T > gpurun_out/r2e_phase_T.json 2>&1
true
