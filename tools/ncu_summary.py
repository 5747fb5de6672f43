"""Summarise an ncu report (raw page) into the metrics the roofline needs.

    python tools/ncu_summary.py gpurun_out/prof_c2.ncu-rep [--json out.json --workload C2 --shape ...]
"""
import csv
import io
import json
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
    "launch__occupancy_limit_shared_mem", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (u, v) for h, u, v in zip(hdr, units, vals)}


def stalls(path, top=12):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, vals = rows[0], rows[2]
    res = []
    for h, v in zip(hdr, vals):
        if h.startswith("smsp__average_warp_latency_issue_stalled_") or \
           (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")):
            try:
                res.append((float(v.replace(",", "")), h))
            except ValueError:
                pass
    return sorted(res, reverse=True)[:top]


def main():
    path = sys.argv[1]
    r = raw(path)
    summ = {}
    for k in WANT:
        if k in r:
            u, v = r[k]
            summ[k] = f"{v} {u}".strip()
    print(json.dumps(summ, indent=1))
    for v, h in stalls(path):
        print(f"  {v:>12.0f}  {h}")
    if "--json" in sys.argv:
        def num(k, scale):
            u, v = r[k]
            return float(v.replace(",", "")) * scale
        mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        rd = num("dram__bytes_read.sum", mult[r["dram__bytes_read.sum"][0]])
        wr = num("dram__bytes_write.sum", mult[r["dram__bytes_write.sum"][0]])
        doc = {"workload": sys.argv[sys.argv.index("--workload") + 1],
               "shape": json.loads(sys.argv[sys.argv.index("--shape") + 1]),
               "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
               "source": path, "metrics": summ}
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
