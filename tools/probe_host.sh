set -x
nproc; free -g; ulimit -l; cat /proc/meminfo | head -5; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; df -h /tmp . | tail -2
python -c "import sys; sys.path.insert(0,'baseline/_ref'); import lfbp; print(lfbp.__file__)"
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu > gpurun_out/p1_c5.json 2> gpurun_out/p1_c5.err; echo rc=$?
cat gpurun_out/p1_c5.json
