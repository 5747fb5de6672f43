"""K1 on the paper's Table 1 geometries (n_z = 11 as in the
table; f32), autotuned plan, against torch copy_ of the same bytes.

    python tools/paper_shapes.py [--secs 0.3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(89, 89, 11, 11), (177, 177, 11, 11), (287, 287, 11, 11), (507, 507, 11, 11), (91, 91, 15, 15),
          (121, 121, 15, 15), (211, 211, 21, 21), (249, 249, 31, 31), (311, 311, 31, 31), (307, 307, 51, 51),
          (181, 181, 95, 55)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--secs", type=float, default=0.3)
    ap.add_argument("--nz", type=int, default=11)
    ap.add_argument("--only", default="", help="comma-separated indices into SHAPES")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device, plan

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
    shapes = [SHAPES[int(i)] for i in a.only.split(",")] if a.only else SHAPES
    for s4 in shapes:
        shape = s4 + (a.nz,)
        src = f_order_empty(shape, torch.float32)
        src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
        out = f_order_empty(shape, torch.float32)
        ms = timed(lambda: hprime_device(src, out=out))
        fs, fo = src.permute(4, 3, 2, 1, 0).reshape(-1), out.permute(4, 3, 2, 1, 0).reshape(-1)
        cms = timed(lambda: fo.copy_(fs))
        nb = 2 * src.numel() * 4
        p = plan(shape)
        print(json.dumps({"tag": a.tag, "shape": shape, "plane_mb": round(src.numel() * 4 / a.nz / 1e6, 1), "ms": round(ms, 4),
                          "GBps": round(nb / ms / 1e6, 1), "copy_GBps": round(nb / cms / 1e6, 1),
                          "frac_of_copy": round(cms / ms, 3), "Gelem_s": round(src.numel() / ms / 1e6, 1),
                          "knobs": p["knobs"], "J": p["J"], "n_chunks": p["n_chunks"]}), flush=True)
        del src, out, fs, fo
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
