#!/bin/bash
# refresh the committed evidence: bench lines, K1 launch list, one full ncu
# capture of the tuned K1 on C2.  The ncu runs pin the plan the headline bench
# run's autotuner chose (env knobs), so no autotuning happens under the
# profiler and the first timed launch is launch index = warmup.
# KN_GIVEN="LFBP_STAGES=.. LFBP_STAGE_KB=.. LFBP_CONSUMER_WARPS=.. LFBP_SUBWARP=.." skips the
# benches and profiles that plan.
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-verify"
if [ -z "$KN_GIVEN" ]; then
  timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
  for c in C1 C3 C4 C5; do
    timeout 600 python bench.py --config $c --steps 50 --no-cpu --no-e2e > gpurun_out/bench_$c.log 2>&1; echo bench_${c}_rc=$?
  done
  KN=$(python -c '
import json; d=json.loads([l for l in open("gpurun_out/bench.log") if l.startswith("{")][-1])
k=d["config"]["kernel_plan"]["knobs"]; print(f"LFBP_STAGES={k[0]} LFBP_STAGE_KB={k[1]} LFBP_CONSUMER_WARPS={k[2]} LFBP_SUBWARP={k[3]}")')
else
  KN="$KN_GIVEN"
fi
echo "pinned plan: $KN" | tee gpurun_out/ncu_plan.txt
env $KN $CMD > gpurun_out/plain_pinned.log 2>&1 && env $KN ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
env $KN ncu --set full --clock-control none --import-source on -k regex:hprime_kernel -s 3 -c 1 -o gpurun_out/prof_c2 -f $CMD > gpurun_out/ncu_c2.log 2>&1; echo ncu2_rc=$?
true
