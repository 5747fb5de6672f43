"""K1 (or copy_) back to back for T seconds in ~50 ms windows: per window the
GB/s (CUDA events), SM clock, power and throttle reasons (NVML).
    python tools/power_trace.py 631,631,21,21,16 [--secs 3] [--op k1|copy] [--tag x]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shape")
    ap.add_argument("--secs", type=float, default=3.0)
    ap.add_argument("--op", default="k1")
    ap.add_argument("--f64", action="store_true")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    import pynvml
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    shape = tuple(int(v) for v in a.shape.split(","))
    dt = torch.float64 if a.f64 else torch.float32
    src = f_order_empty(shape, dt)
    src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
    out = f_order_empty(shape, dt)
    nbytes = src.numel() * src.element_size()
    flat_s, flat_o = src.permute(4, 3, 2, 1, 0).reshape(-1), out.permute(4, 3, 2, 1, 0).reshape(-1)

    def op():
        if a.op == "k1":
            hprime_device(src, out=out)
        else:
            flat_o.copy_(flat_s)

    op()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    op()
    e1.record()
    torch.cuda.synchronize()
    per = max(1, int(50.0 / e0.elapsed_time(e1)))
    rows = []
    t_total = 0.0
    while t_total < a.secs * 1e3:
        e0.record()
        for _ in range(per):
            op()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        t_total += ms
        clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        rows.append([round(t_total, 1), round(2 * nbytes * per / ms / 1e6, 1), clk, round(pw, 1), hex(rs)])
    print(json.dumps({"tag": a.tag, "op": a.op, "lib": os.environ.get("LFBP_LIB_PATH", "in-tree"),
                      "shape": shape, "per_window": per, "rows": rows}), flush=True)


if __name__ == "__main__":
    main()
