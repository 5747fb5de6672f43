"""Run-to-run stability of K1 plans: interleaved repeats of a few plans.
    python tools/stability.py --config C2 --plans "3,48,16,16;4,48,16,16;3,48,8,8" --rounds 5 --reps 200
A plan is stages,stage_kb,consumer_warps,sub_width[,kflags (LFBP_KFLAGS)].
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
    ap.add_argument("--plans", default="3,48,16,16;4,48,16,16;3,48,8,8")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=200)
    a = ap.parse_args()
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device
    from paper_2003_09133_b200.configs import WORKLOADS
    w = WORKLOADS[a.config]
    tdt = torch.float32 if w.itemsize == 4 else torch.float64
    src = f_order_empty(w.shape, tdt)
    src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
    out = f_order_empty(w.shape, tdt)
    keys = ("LFBP_STAGES", "LFBP_STAGE_KB", "LFBP_CONSUMER_WARPS", "LFBP_SUBWARP", "LFBP_KFLAGS")
    plans = [tuple(int(v) for v in p.split(",")) for p in a.plans.split(";")]
    res = {p: [] for p in plans}
    for r in range(a.rounds):
        for pl in plans:
            for k, v in zip(keys, list(pl) + [""] * len(keys)):
                os.environ[k] = str(v)
            for _ in range(5):
                hprime_device(src, out=out)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.reps):
                hprime_device(src, out=out)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            res[pl].append(round(2 * w.nbytes / ms / 1e6, 1))
    for pl, v in res.items():
        print(json.dumps({"config": a.config, "plan": pl, "GBps": v}), flush=True)


if __name__ == "__main__":
    main()
