"""Kernel tuning sweep on the GPU box (timing only; parity lives in tests/).

    python tools/sweep.py --configs C2,C4,181x181x95x55x11 [--grid default|wide] [--reps 20]

Inputs are filled on the device (torch.rand) -- values do not affect a copy
kernel.  The plan knobs are environment variables read by the C-ABI planner
on every call (LFBP_STAGES, LFBP_STAGE_KB, LFBP_CONSUMER_WARPS,
LFBP_CTAS_PER_SM, LFBP_PITCH_EXTRA16).  Prints one JSON line per variant.
"""
from __future__ import annotations

import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2")
    ap.add_argument("--grid", default="default")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device, plan
    from paper_2003_09133_b200.configs import WORKLOADS
    peak = 6542.1
    if a.grid == "default":
        a.grid = "STAGES=3,4,6;STAGE_KB=16,24,32;CONSUMER_WARPS=4,8,16;CTAS_PER_SM=0,2"
    spec = [kv.split("=") for kv in a.grid.split(";")]
    keys = tuple("LFBP_" + k for k, _ in spec)
    grid = list(itertools.product(*[[int(v) for v in vs.split(",")] for _, vs in spec]))
    class _Shape:  # "181x181x95x55x11" (f32) instead of a BASELINE config name
        def __init__(self, spec):
            import numpy as np
            self.shape = tuple(int(v) for v in spec.split("x"))
            self.dtype = np.float32
            self.itemsize = 4
            self.nbytes = int(np.prod(self.shape)) * 4

    for cfg in a.configs.split(","):
        w = WORKLOADS[cfg] if cfg in WORKLOADS else _Shape(cfg)
        tdt = torch.float32 if w.itemsize == 4 else torch.float64
        src = f_order_empty(w.shape, tdt)
        src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
        out = f_order_empty(w.shape, tdt)
        nbytes = 2 * w.nbytes
        best = None
        for combo in grid:
            for k, v in zip(keys, combo):
                if v or k == "LFBP_KFLAGS":
                    os.environ[k] = str(v)
                else:
                    os.environ.pop(k, None)
            try:
                p = plan(w.shape, w.dtype)
                for _ in range(3):
                    hprime_device(src, out=out)
                torch.cuda.synchronize()
                # time >= ~60 ms per variant (short windows are biased by clock / power transients)
                t0 = torch.cuda.Event(enable_timing=True)
                t1 = torch.cuda.Event(enable_timing=True)
                t0.record()
                hprime_device(src, out=out)
                t1.record()
                torch.cuda.synchronize()
                reps = max(a.reps, int(60.0 / max(t0.elapsed_time(t1), 1e-3)))
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    hprime_device(src, out=out)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
            except Exception as exc:  # noqa: BLE001
                print(json.dumps({"config": cfg, "knobs": combo, "error": str(exc)}), flush=True)
                continue
            gbs = nbytes / ms / 1e6
            rec = {"config": cfg, "knobs": dict(zip(keys, combo)), "ms": round(ms, 4), "GBps": round(gbs, 1),
                   "frac": round(gbs / peak, 4), "plan": {k: p[k] for k in ("J", "stages", "threads", "ctas_per_sm",
                                                                         "stage_bytes", "grid")}}
            print(json.dumps(rec), flush=True)
            if best is None or gbs > best["GBps"]:
                best = rec
        for k in keys:
            os.environ.pop(k, None)
        print(json.dumps({"best": best}), flush=True)
        del src, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
