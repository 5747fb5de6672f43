#!/bin/bash
# (1) the HP_CHECKED build under fuzz and parity tests (rerun: smem reserve fix);
# (2) broad plan sweep on C2 / C3 (row consumer and task consumer, static and
#     dynamic tickets) to find candidates for their per-SM-bound rates.
mkdir -p gpurun_out; L=gpurun_out/r2q.log; : > $L
CK=abtest/libhprime_CHECKED.so
for f in 0 32 128 200; do
  LFBP_LIB_PATH=$CK LFBP_KFLAGS=$f LFBP_ZCHUNK_MB=1 timeout 900 python tools/fuzz_parity.py --cases 150 --seed $((21 + f)) > gpurun_out/r2q_fuzz_$f.log 2>&1
  echo "checked fuzz flags=$f rc=$?" >> $L; tail -1 gpurun_out/r2q_fuzz_$f.log >> $L
done
LFBP_LIB_PATH=$CK timeout 1800 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "unit_orders or plan_variants or random_shapes or golden or z_range or unaligned" > gpurun_out/r2q_checked_pytest.log 2>&1
echo "checked pytest rc=$?" >> $L; tail -1 gpurun_out/r2q_checked_pytest.log >> $L
timeout 1200 python tools/sweep.py --configs C3,C2 --grid "STAGES=2,3,4,6;STAGE_KB=32,48,64,96,128;CONSUMER_WARPS=8,12,16;SUBWARP=8,16,32;KFLAGS=0,128" > gpurun_out/r2q_sweep_row.jsonl 2>&1
echo "sweep row rc=$?" >> $L
timeout 900 python tools/sweep.py --configs C3,C2 --grid "STAGES=2,3,4,6;STAGE_KB=32,48,64,96,128;CONSUMER_WARPS=8,12,16;KFLAGS=32,160" > gpurun_out/r2q_sweep_tasks.jsonl 2>&1
echo "sweep tasks rc=$?" >> $L
true
