#!/bin/bash
mkdir -p gpurun_out
run() {  # name config envs...
  local name=$1 cfg=$2; shift 2
  local CMD="python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu --no-e2e --no-verify"
  env "$@" $CMD > gpurun_out/plain_$name.log 2>&1 && \
  env "$@" ncu --set full --clock-control none --import-source on -k regex:hprime_kernel -s 3 -c 1 -o gpurun_out/prof_$name -f $CMD > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
}
run c3b C3 LFBP_STAGES=4 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=16
run c2b C2 LFBP_STAGES=3 LFBP_STAGE_KB=48 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=8
true
