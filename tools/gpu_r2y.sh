#!/bin/bash
# e2e ceiling: pinned PCIe rates (plane-sized chunks of C5 and C2) and the
# per-chunk timeline of the C5 host pipeline
mkdir -p gpurun_out
timeout 600 python tools/pcie_probe.py --mb 14000 --chunk-mb 702 > gpurun_out/r2y_pcie_c5.jsonl 2>&1
timeout 600 python tools/pcie_probe.py --mb 1745 --chunk-mb 34 > gpurun_out/r2y_pcie_c2.jsonl 2>&1
LFBP_TRACE=1 timeout 900 python tools/e2e_trace.py --config C5 > gpurun_out/r2y_trace_c5.out 2> gpurun_out/r2y_trace_c5.txt
echo "trace rc=$?" >> gpurun_out/r2y_trace_c5.out
true
