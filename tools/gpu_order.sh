mkdir -p gpurun_out
o=gpurun_out/bigshape_order.jsonl; : > $o
for kf in 0 4; do
timeout 300 python tools/tlb_probe.py --base 181,181,95 --ny 55 --gb 15 --plan 4,48,8,8 --kflags $kf --secs 0.3 >> $o 2>&1
timeout 300 python tools/tlb_probe.py --base 307,307,51 --ny 51 --gb 21 --plan 4,48,8,16 --kflags $kf --secs 0.3 >> $o 2>&1
timeout 300 python tools/tlb_probe.py --base 195,195,15 --ny 15 --plan 3,48,8,8 --kflags $kf --secs 0.3 >> $o 2>&1
done
