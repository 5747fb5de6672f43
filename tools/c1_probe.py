"""C1 (26 MB moved, latency-bound): K1 against torch copy_ of the same bytes
and an (almost) empty launch, timed exactly like bench.py times C1 (per-step
CUDA events around the launch, 512 MB L2 flush write between steps), and
again with L2 left warm.  Gives the achievable floor at this size.

    python tools/c1_probe.py [--steps 200] [--config C1]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--config", default="C1")
    a = ap.parse_args()
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device, plan
    from paper_2003_09133_b200.configs import WORKLOADS
    w = WORKLOADS[a.config]
    tdt = torch.float32 if w.itemsize == 4 else torch.float64
    src = f_order_empty(w.shape, tdt)
    src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
    out = f_order_empty(w.shape, tdt)
    fs, fo = src.permute(4, 3, 2, 1, 0).reshape(-1), out.permute(4, 3, 2, 1, 0).reshape(-1)
    tiny = torch.empty(1, dtype=torch.float32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    nb = 2 * w.nbytes
    arms = {"k1": lambda: hprime_device(src, out=out), "copy": lambda: fo.copy_(fs),
            "empty": lambda: tiny.fill_(0.0)}
    for fn in arms.values():
        for _ in range(5):
            fn()
    torch.cuda.synchronize()
    for flushed in (True, False):
        for name, fn in arms.items():
            st = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
            en = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
            for k in range(a.steps):
                if flushed:
                    flush.fill_(k & 0xff)
                st[k].record()
                fn()
                en[k].record()
            torch.cuda.synchronize()
            ms = [s.elapsed_time(e) for s, e in zip(st, en)]
            avg = statistics.mean(ms)
            print(json.dumps({"config": a.config, "arm": name, "l2_flushed": flushed, "us_avg": round(avg * 1e3, 2),
                              "us_median": round(statistics.median(ms) * 1e3, 2),
                              "us_min": round(min(ms) * 1e3, 2),
                              "GBps": round(nb / (avg * 1e-3) / 1e9, 1) if name != "empty" else None}), flush=True)
    print(json.dumps({"plan": plan(w.shape, w.dtype)}), flush=True)


if __name__ == "__main__":
    main()
