#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "cphase" > gpurun_out/cp2_tests.log 2>&1
echo "rc=$?" >> gpurun_out/cp2_tests.log
o=gpurun_out/cp2.jsonl; : > $o
K="LFBP_AUTOTUNE=0 LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32"
for f in 88 24; do
  env $K LFBP_KFLAGS=$f timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 40 --gap 2 --tag C5_f$f >> $o 2>&1; sleep 3
done
env $K LFBP_KFLAGS=88 LFBP_CONSUMER_WARPS=4 timeout 300 python tools/phase_trace.py 631,631,21,21,101 --bursts 1 --launches 40 --gap 2 --tag C5_f88_w4 >> $o 2>&1
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_short_scoreboard,smsp__pcsamp_warps_issue_stalled_wait,smsp__pcsamp_warps_issue_stalled_barrier,smsp__pcsamp_warps_issue_stalled_membar,smsp__pcsamp_warps_issue_stalled_lg_throttle,smsp__pcsamp_warps_issue_stalled_mio_throttle,smsp__pcsamp_warps_issue_stalled_drain,smsp__pcsamp_warps_issue_stalled_selected,smsp__pcsamp_warps_issue_stalled_sleeping,smsp__pcsamp_warps_issue_stalled_branch_resolving
for f in 88 24; do
env $K LFBP_KFLAGS=$f timeout 600 ncu --clock-control none --metrics $M -k regex:hprime_kernel -s 1 -c 1 --csv python tools/ncu_one.py 631,631,21,21,8 > gpurun_out/ncu_cp_f$f.csv 2>&1
done
true
