"""Two K1 launches on one shape (fixed plan from LFBP_* env) for ncu
captures of the second: python tools/ncu_one.py 631,631,21,21,101"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device
    shape = tuple(int(v) for v in sys.argv[1].split(","))
    dt = torch.float64 if "--f64" in sys.argv else torch.float32
    src = f_order_empty(shape, dt)
    src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
    out = f_order_empty(shape, dt)
    for _ in range(2):
        hprime_device(src, out=out)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
