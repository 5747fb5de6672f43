"""K1 over a whole array as ONE launch against the same planes as several
z-chunk launches back to back (same plan from LFBP_* env): does the rate of
long launches fall because persistent CTAs drift apart over time?
    python tools/zchunk_probe.py 631,631,21,21,101 --chunks 0,8,16,26,51 [--reps 5]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shape")
    ap.add_argument("--chunks", default="0,8,16,26,51")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device
    shape = tuple(int(v) for v in a.shape.split(","))
    src = f_order_empty(shape, torch.float32)
    src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
    out = f_order_empty(shape, torch.float32)
    nbytes = src.numel() * 4
    nz = shape[4]

    def run(k):
        if k == 0 or k >= nz:
            hprime_device(src, out=out)
        else:
            for z0 in range(0, nz, k):
                hprime_device(src, out=out, z_range=(z0, min(nz, z0 + k)))

    res = {}
    ks = [int(v) for v in a.chunks.split(",")]
    for k in ks:
        run(k)
    torch.cuda.synchronize()
    for _ in range(a.rounds):
        for k in ks:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                run(k)
            e1.record()
            torch.cuda.synchronize()
            res.setdefault(k, []).append(round(2 * nbytes * a.reps / e0.elapsed_time(e1) / 1e6, 1))
    print(json.dumps({"tag": a.tag, "shape": shape, "env": {k: v for k, v in os.environ.items() if k.startswith("LFBP_")},
                      "GBps_by_chunk_planes": res}), flush=True)


if __name__ == "__main__":
    main()
