#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) on the small K1 probe
# (every consumer / scheduling variant), then the C5 drop-in on host arrays.
mkdir -p gpurun_out; L=gpurun_out/r2o.log; : > $L
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_probe.py > gpurun_out/r2o_san_$t.log 2>&1
  echo "sanitizer $t rc=$?" >> $L; tail -3 gpurun_out/r2o_san_$t.log >> $L
done
timeout 1800 python tools/c5_dropin.py > gpurun_out/r2o_c5_dropin.json 2> gpurun_out/r2o_c5_dropin.err
echo "c5 dropin rc=$?" >> $L
true
