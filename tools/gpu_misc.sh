#!/bin/bash
# C1 latency, the torchrun (NCCL) code path on one GPU, the K1 launch list
mkdir -p gpurun_out
timeout 420 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python bench.py --config C1 --steps 50 --no-cpu --no-e2e > gpurun_out/bench_C1.log 2>&1; echo c1_rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/bench_torchrun1.log 2>&1; echo trun_rc=$?
timeout 300 python bench.py --config C3 --strong --steps 10 --no-cpu --no-e2e > gpurun_out/bench_C3_strong.log 2>&1; echo c3s_rc=$?
CMD="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-verify"
$CMD > gpurun_out/plain_launch.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?
true
