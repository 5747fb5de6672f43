#!/bin/bash
# (1) the HP_CHECKED build (bounds + ring-protocol checks, the stand-in for
#     compute-sanitizer, which the pool has closed) under the fuzz sweep and
#     the plan / order / random-shape parity tests;
# (2) mbarrier wait with a suspend-time hint: A/B of library builds.
mkdir -p gpurun_out; L=gpurun_out/r2p.log; : > $L
CK=abtest/libhprime_CHECKED.so
for f in 0 32 128 200; do
  LFBP_LIB_PATH=$CK LFBP_KFLAGS=$f LFBP_ZCHUNK_MB=1 timeout 900 python tools/fuzz_parity.py --cases 150 --seed $((21 + f)) > gpurun_out/r2p_fuzz_$f.log 2>&1
  echo "checked fuzz flags=$f rc=$?" >> $L; tail -1 gpurun_out/r2p_fuzz_$f.log >> $L
done
LFBP_LIB_PATH=$CK timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "unit_orders or plan_variants or random_shapes or golden or z_range or unaligned" > gpurun_out/r2p_checked_pytest.log 2>&1
echo "checked pytest rc=$?" >> $L; tail -1 gpurun_out/r2p_checked_pytest.log >> $L
o=gpurun_out/r2p.jsonl; : > $o
for rep in 1 2; do
for lib in BASE HINT20K HINT1M; do
  LFBP_LIB_PATH=abtest/libhprime_$lib.so timeout 300 python tools/k1_probe.py 631,631,21,21,101 --reps 10 --tag C5_$lib >> $o 2>&1
  LFBP_LIB_PATH=abtest/libhprime_$lib.so timeout 300 python tools/k1_probe.py 399,399,19,19,64 --tag C3_$lib >> $o 2>&1
  LFBP_LIB_PATH=abtest/libhprime_$lib.so timeout 300 python tools/k1_probe.py 195,195,15,15,51 --reps 100 --tag C2_$lib >> $o 2>&1
done
done
true
