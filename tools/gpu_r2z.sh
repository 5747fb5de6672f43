#!/bin/bash
# final fuzz campaign: random plans incl. the kernel options of the tuned
# plans, and the checked build with the shipped ticket flags forced
mkdir -p gpurun_out; L=gpurun_out/r2z.log; : > $L
[ -f abtest/libhprime_CHECKED.so ] || tools/build_variant.sh CHECKED -DHP_CHECKED
timeout 1800 python tools/fuzz_parity.py --cases 1500 --seed 2026 > gpurun_out/r2z_fuzz_default.log 2>&1
echo "default rc=$?" >> $L; tail -1 gpurun_out/r2z_fuzz_default.log >> $L
LFBP_LIB_PATH=abtest/libhprime_CHECKED.so LFBP_KFLAGS=136 timeout 1800 python tools/fuzz_parity.py --cases 800 --seed 2027 > gpurun_out/r2z_fuzz_checked136.log 2>&1
echo "checked136 rc=$?" >> $L; tail -1 gpurun_out/r2z_fuzz_checked136.log >> $L
LFBP_LIB_PATH=abtest/libhprime_CHECKED.so LFBP_KFLAGS=160 timeout 1800 python tools/fuzz_parity.py --cases 400 --seed 2028 > gpurun_out/r2z_fuzz_checked160.log 2>&1
echo "checked160 rc=$?" >> $L; tail -1 gpurun_out/r2z_fuzz_checked160.log >> $L
true
