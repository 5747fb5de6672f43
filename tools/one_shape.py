"""Run K1 a few times on one shape (for ncu captures).
    python tools/one_shape.py 181,181,95,55,11 [--reps 3]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shape")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device, plan
    shape = tuple(int(v) for v in a.shape.split(","))
    src = f_order_empty(shape, torch.float32)
    src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
    out = f_order_empty(shape, torch.float32)
    for _ in range(a.reps):
        hprime_device(src, out=out)
    torch.cuda.synchronize()
    print(plan(shape))


if __name__ == "__main__":
    main()
