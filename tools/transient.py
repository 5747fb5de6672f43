"""How long does K1 take to reach its steady rate after a plan switch?
Runs a sequence of plans, each for --windows windows of --reps launches,
and prints every window's GB/s.

    python tools/transient.py --config C2 --seq "4,48,16,16;4,48,8,8;2,96,8,8;4,48,8,8"
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--seq", default="4,48,16,16;4,48,8,8;2,96,8,8;4,48,8,8")
    ap.add_argument("--windows", type=int, default=12)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--sep", default="none", choices=["none", "tiny", "flush"],
                    help="between launches: nothing (back to back), a 1-element fill, or a 256 MB fill")
    a = ap.parse_args()
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device
    from paper_2003_09133_b200.configs import WORKLOADS
    w = WORKLOADS[a.config]
    tdt = torch.float32 if w.itemsize == 4 else torch.float64
    src = f_order_empty(w.shape, tdt)
    src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
    out = f_order_empty(w.shape, tdt)
    tiny = torch.empty(1 if a.sep == "tiny" else (256 << 20), dtype=torch.uint8, device="cuda")
    keys = ("LFBP_STAGES", "LFBP_STAGE_KB", "LFBP_CONSUMER_WARPS", "LFBP_SUBWARP", "LFBP_KFLAGS")
    for pl in a.seq.split(";"):
        for k, v in zip(keys, pl.split(",") + [""] * len(keys)):
            os.environ[k] = v
        if a.sep == "none":
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.windows + 1)]
            torch.cuda.synchronize()
            ev[0].record()
            for i in range(a.windows):
                for _ in range(a.reps):
                    hprime_device(src, out=out)
                ev[i + 1].record()
            torch.cuda.synchronize()
            rates = [round(2 * w.nbytes * a.reps / ev[i].elapsed_time(ev[i + 1]) / 1e6, 1) for i in range(a.windows)]
        else:  # per-launch events, a separating kernel outside them
            n = a.windows * a.reps
            st = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
            en = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
            torch.cuda.synchronize()
            for k in range(n):
                tiny.fill_(k & 0xff)
                st[k].record()
                hprime_device(src, out=out)
                en[k].record()
            torch.cuda.synchronize()
            ms = [s_.elapsed_time(e_) for s_, e_ in zip(st, en)]
            rates = [round(2 * w.nbytes * a.reps / sum(ms[i * a.reps:(i + 1) * a.reps]) / 1e6, 1)
                     for i in range(a.windows)]
        print(json.dumps({"config": a.config, "plan": pl, "sep": a.sep, "GBps_per_window": rates}), flush=True)


if __name__ == "__main__":
    main()
