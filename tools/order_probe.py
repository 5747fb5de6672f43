"""Unit-order probe: K1 on one shape with y blocks of different heights
(LFBP_TILE_Y; n_y = plain y-fastest order), interleaved rounds, against
torch copy_ of the same bytes.

    python tools/order_probe.py 181,181,95,55,11 --tiles 55,4,8,12,16 [--plan 2,96,8,8] [--f64]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shape")
    ap.add_argument("--tiles", default="")
    ap.add_argument("--plan", default="")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--secs", type=float, default=0.15)
    ap.add_argument("--f64", action="store_true")
    a = ap.parse_args()
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device, plan
    shape = tuple(int(v) for v in a.shape.split(","))
    if a.plan:
        for k, v in zip(("LFBP_STAGES", "LFBP_STAGE_KB", "LFBP_CONSUMER_WARPS", "LFBP_SUBWARP"), a.plan.split(",")):
            os.environ[k] = v
    tdt = torch.float64 if a.f64 else torch.float32
    src = f_order_empty(shape, tdt)
    src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
    out = f_order_empty(shape, tdt)
    nbytes = 2 * src.numel() * src.element_size()
    tiles = [int(v) for v in a.tiles.split(",")] if a.tiles else [shape[3]]

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        reps = max(3, int(a.secs * 1e3 / max(e0.elapsed_time(e1), 1e-3)))
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    fs, fo = src.permute(4, 3, 2, 1, 0).reshape(-1), out.permute(4, 3, 2, 1, 0).reshape(-1)
    res = {t: [] for t in tiles}
    copy = []
    for _ in range(a.rounds):
        for t in tiles:
            os.environ["LFBP_TILE_Y"] = str(t)
            res[t].append(round(nbytes / timed(lambda: hprime_device(src, out=out)) / 1e6, 1))
        copy.append(round(nbytes / timed(lambda: fo.copy_(fs)) / 1e6, 1))
    p = plan(shape, "float64" if a.f64 else "float32")
    for t in tiles:
        best = max(res[t])
        print(json.dumps({"shape": shape, "tile_y": t, "GBps": res[t], "frac_of_copy": round(best / max(copy), 3),
                          "copy_GBps": copy, "knobs": p["knobs"], "J": p["J"]}), flush=True)


if __name__ == "__main__":
    main()
