#!/bin/bash
# y-block unit order (LFBP_TILE_Y) on large-n_y shapes and the BASELINE configs
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "plan_variants or random_shapes or randomised" --timeout 600 > gpurun_out/pytest_order.log 2>&1; echo parity_rc=$? | tee -a gpurun_out/pytest_order.log
o=gpurun_out/order_probe.jsonl; : > $o
timeout 300 python tools/order_probe.py 181,181,95,55,11 --tiles 55,4,8,12,16,24 --plan 2,96,8,8 >> $o 2>&1
timeout 300 python tools/order_probe.py 307,307,51,51,11 --tiles 51,4,8,12,16,24 --plan 2,96,8,8 >> $o 2>&1
timeout 300 python tools/order_probe.py 249,249,31,31,11 --tiles 31,4,8,12,16 --plan 2,96,8,8 >> $o 2>&1
timeout 300 python tools/order_probe.py 195,195,15,121,14 --tiles 121,8,15,24,32 --plan 4,48,8,8 >> $o 2>&1
timeout 300 python tools/order_probe.py 195,195,15,15,51 --tiles 15,4,8 --plan 4,48,8,8 >> $o 2>&1
timeout 300 python tools/order_probe.py 631,631,21,21,16 --tiles 21,3,7,11 --plan 3,64,8,32 >> $o 2>&1
timeout 300 python tools/order_probe.py 399,399,19,19,32 --tiles 19,5,10 --plan 2,96,8,16 >> $o 2>&1
timeout 300 python tools/order_probe.py 273,273,13,13,41 --tiles 13,4,7 --plan 4,48,8,16 --f64 >> $o 2>&1
true
