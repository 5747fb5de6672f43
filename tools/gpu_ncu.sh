#!/bin/bash
# ncu full captures of K1 at the tuned plans (each command first runs clean without ncu)
mkdir -p gpurun_out
run() {  # name config envs...
  local name=$1 cfg=$2; shift 2
  local CMD="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-e2e --no-verify"
  env "$@" $CMD > gpurun_out/plain_$name.log 2>&1 && \
  env "$@" ncu --set full --clock-control none --import-source on -k regex:hprime_kernel -s 3 -c 1 -o gpurun_out/prof_$name -f $CMD > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
}
run c2 C2 LFBP_STAGES=3 LFBP_STAGE_KB=32 LFBP_CONSUMER_WARPS=8
run c3 C3 LFBP_STAGES=3 LFBP_STAGE_KB=16 LFBP_CONSUMER_WARPS=6
run c4 C4 LFBP_STAGES=3 LFBP_STAGE_KB=32 LFBP_CONSUMER_WARPS=4
