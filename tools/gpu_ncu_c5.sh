#!/bin/bash
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__cycles_active_read.sum,dram__cycles_active_write.sum,dram__cycles_elapsed.avg,lts__d_sectors_fill_device.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,lts__t_requests_op_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_write.sum
K="LFBP_AUTOTUNE=0 LFBP_STAGES=3 LFBP_STAGE_KB=64 LFBP_CONSUMER_WARPS=8 LFBP_SUBWARP=32"
for v in "f0:LFBP_KFLAGS=0" "f8:LFBP_KFLAGS=8" "f8g140:LFBP_KFLAGS=8 LFBP_GRID=140"; do
  tag=${v%%:*}; e=${v#*:}
  env $K $e timeout 900 ncu --replay-mode application --clock-control none --metrics $M -k regex:hprime_kernel -s 1 -c 1 --csv python tools/ncu_one.py 631,631,21,21,101 > gpurun_out/ncu_c5_$tag.csv 2> gpurun_out/ncu_c5_$tag.err
  env $K $e timeout 900 ncu --replay-mode application --clock-control none --metrics $M -k regex:hprime_kernel -s 1 -c 1 --csv python tools/ncu_one.py 631,631,21,21,16 > gpurun_out/ncu_c5s16_$tag.csv 2> gpurun_out/ncu_c5s16_$tag.err
done
true
