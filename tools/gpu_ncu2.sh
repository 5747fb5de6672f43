#!/bin/bash
# ncu full captures of K1 for C3 and C5 at their best swept plans
mkdir -p gpurun_out
run() {  # name config envs...
  local name=$1 cfg=$2; shift 2
  local CMD="python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu --no-e2e --no-verify"
  env "$@" $CMD > gpurun_out/plain_$name.log 2>&1 && \
  env "$@" ncu --set full --clock-control none --import-source on -k regex:hprime_kernel -s 3 -c 1 -o gpurun_out/prof_$name -f $CMD > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
}
run c3 C3 LFBP_STAGES=4 LFBP_STAGE_KB=32 LFBP_CONSUMER_WARPS=16 LFBP_SUBWARP=32
run c5 C5 LFBP_STAGES=4 LFBP_STAGE_KB=32 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32
run c4 C4 LFBP_STAGES=4 LFBP_STAGE_KB=32 LFBP_CONSUMER_WARPS=12 LFBP_SUBWARP=32
true
