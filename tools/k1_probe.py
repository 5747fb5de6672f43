"""Time K1 on one shape with the autotuned plan (or LFBP_* knobs), interleaved
rounds; for same-box A/B of library builds (LFBP_LIB_PATH) and debug builds.
    python tools/k1_probe.py 631,631,21,21,16 [--reps 20] [--rounds 3] [--f64]"""
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
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--f64", action="store_true")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device, plan
    shape = tuple(int(v) for v in a.shape.split(","))
    dt = torch.float64 if a.f64 else torch.float32
    src = f_order_empty(shape, dt)
    src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
    out = f_order_empty(shape, dt)
    nbytes = src.numel() * src.element_size()
    for _ in range(3):
        hprime_device(src, out=out)
    torch.cuda.synchronize()
    res = []
    for _ in range(a.rounds):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            hprime_device(src, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        res.append(round(2 * nbytes / ms / 1e6, 1))
    print(json.dumps({"tag": a.tag, "lib": os.environ.get("LFBP_LIB_PATH", "in-tree"), "shape": shape,
                      "GBps_rw": res, "plan": plan(shape, np.float64 if a.f64 else np.float32)}), flush=True)


if __name__ == "__main__":
    main()
